// Activation swap engine (fy_swapper_*): the GPU -> pinned host (-> SSD)
// copy path of the reference's activation swap tasks, as a component a
// training framework calls directly (the graph executor runs the same
// legs inside offsim_execute).
//
//   swap out, placement CPU   D2H into NUMA-local pinned memory
//   swap out, placement SSD   D2H into a bounded ring of pinned slots, each
//                             slot written to an O_DIRECT file through the
//                             io_uring engine as soon as it lands
//   swap in                   the reverse legs; SSD pieces are read into the
//                             ring and copied H2D slot by slot
//
// Reference tasks: `fwd act_g2c / act_c2s`, `fwd ckpt_g2c / ckpt_c2s`
// (proj/src/task_graph.cpp:296-321) and `bwd ckpt_s2c / ckpt_c2g`,
// `bwd act_s2c / act_c2g` (:357-397); placement = the planner's
// checkpoint_location (proj/src/runner.cpp:90-106).
//
// Everything is stream-ordered: copies on two copy streams, file IO as host
// functions on a third stream, slot reuse and handle completion as CUDA
// events, so calls return as soon as the work is enqueued.
#pragma once

#include "../core/io_engine.hpp"
#include "fuyou/fy_adam.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace fy {

class Swapper {
public:
    explicit Swapper(const fy_swap_config& cfg);
    ~Swapper();
    Swapper(const Swapper&) = delete;
    Swapper& operator=(const Swapper&) = delete;

    std::uint64_t swap_out(const void* src, std::uint64_t bytes, int placement, cudaEvent_t ready,
                           cudaEvent_t src_free);
    void swap_in(std::uint64_t handle, void* dst, cudaEvent_t ready, cudaEvent_t done);
    void release(std::uint64_t handle);
    void sync();
    std::uint64_t host_bytes() const { return host_bytes_; }
    std::uint64_t file_bytes() const { return file_end_; }
    const char* io_engine() const { return io_.engine(); }

    struct IoReq {
        Swapper* self;
        void* buf;
        std::uint64_t bytes;
        std::uint64_t offset;
        bool write;
    };

private:
    struct Entry {
        std::uint64_t bytes = 0;
        int placement = FY_SWAP_CPU;
        void* host = nullptr;          // CPU placement
        std::uint64_t host_cap = 0;
        std::uint64_t file_off = 0;    // SSD placement
        cudaEvent_t stored = nullptr;  // data complete in its tier
    };
    void* take_host(std::uint64_t bytes, std::uint64_t* cap);
    void give_host(void* p, std::uint64_t cap);
    void open_file();
    void close_files() noexcept;
    void release_all() noexcept;

    fy_swap_config cfg_{};
    std::vector<std::string> dirs_; // one per device (striped when > 1)
    cudaStream_t d2h_ = nullptr, h2d_ = nullptr, io_s_ = nullptr;
    IoEngine io_;
    std::vector<int> fds_;
    std::vector<std::string> paths_;
    std::uint64_t file_end_ = 0;
    std::vector<void*> slots_;
    std::vector<cudaEvent_t> slot_free_, slot_filled_;
    std::uint32_t next_slot_ = 0;
    std::map<std::uint64_t, Entry> entries_;
    std::uint64_t next_handle_ = 1;
    std::multimap<std::uint64_t, void*> free_host_;  // capacity -> pinned buffer
    std::uint64_t host_bytes_ = 0;
    std::deque<IoReq> reqs_;  // stable storage for queued host-function IO

public:
    std::atomic<int> io_failed{0};
    // Released by every IO host function when it finishes and acquired after
    // the stream synchronisations that wait for them: makes the ordering the
    // CUDA runtime guarantees explicit in the C++ memory model (and visible
    // to ThreadSanitizer, which cannot see inside libcuda).
    std::atomic<std::uint64_t> io_done{0};
    std::mutex io_mu;
    std::string io_error;
    IoEngine& engine() { return io_; }
    IoEngine::Stripe stripe() const {
        return {fds_.data(), static_cast<unsigned>(fds_.size()), 4ull << 20};
    }
};

} // namespace fy
