// Sharded optimizer step over the GPUs of one node: the
// reference's optimizer group block (proj/src/task_graph.cpp:453-503) with
// every block split by parameter slice across `world` ranks, one process (or
// one ShardGroup) per GPU, followed by the all-gather of the updated 16-bit
// params — the only exchange the step has.
//
//   per chunk c, rank r       own slice [off_c(r), off_c(r)+count_c(r)) of the
//                             chunk (fy_shard_range, 8-element aligned)
//   states                    caller-owned [master|m|v] of the slice: device
//                             (resident tier) or NUMA-local pinned host
//                             memory streamed through a ChunkPipeline
//   params                    library-owned ARENA: every chunk's full params,
//                             slice-padded (world x stride_c elements), so the
//                             all-gather is in place
//   gather                    NCCL: ncclAllGather per chunk on a comm stream,
//                             started when the chunk's slice is updated;
//                             PEER: the update kernel's epilogue stores every
//                             param into every peer's arena over NVLink
//                             (resident) / the copy engines push the slice
//                             (streamed), peers' arenas mapped by CUDA IPC
//                             or pointers, with device-side entry / exit
//                             barriers (flags in the arenas' headers)
//   grad norm                 the global sum of squares: ncclAllReduce of one
//                             double, or exchanged through the arena headers
//                             in the exit barrier and summed in rank order
#pragma once

#include "adamw_kernels.cuh"
#include "fuyou/fy_adam.h"
#include "pipeline.cuh"

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace fy {

constexpr std::uint32_t kMaxWorld = kMaxPeers + 1;

// Arena header: barrier flags and the per-rank norm / non-finite slots that
// peers write into (4 KiB, then the chunks' param regions, 256-B aligned).
struct ArenaHeader {
    unsigned long long flags[2][kMaxWorld];  // [entry|exit][writer rank] = step sequence
    double norms[kMaxWorld];
    int nonfinite[kMaxWorld];
};
constexpr std::uint64_t kArenaHeaderBytes = 4096;

class ShardGroup {
public:
    explicit ShardGroup(const fy_shard_config& cfg);
    ~ShardGroup();
    ShardGroup(const ShardGroup&) = delete;
    ShardGroup& operator=(const ShardGroup&) = delete;

    void slice_info(std::uint32_t chunk, fy_shard_slice* out) const;
    void ipc_handle(void* out) const;
    void connect_handles(const void* handles);       // world x FY_IPC_HANDLE_BYTES
    void connect_ptrs(void* const* arenas);          // world arena base pointers
    void step(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm, cudaStream_t stream);
    void wait(double* grad_sq_sum, int* nonfinite);
    void stats(fy_shard_stats* out) const;
    // per chunk of the last step: device time of its update kernel(s), ms
    void update_ms(double* out, std::uint32_t count) const;
    void* arena() const { return arena_; }
    std::uint64_t arena_bytes() const { return arena_bytes_; }

private:
    struct Slice {
        std::uint64_t n = 0, offset = 0, count = 0, stride = 0;
        std::uint64_t arena_off = 0;  // bytes from the arena base to the chunk's region
    };
    void release() noexcept;
    void need_connected() const;
    // device-side barrier over the peers' arena headers; with my_norm the
    // exit barrier also exchanges the per-rank sums / flags (into d_total_)
    void barrier(int kind, cudaStream_t s, const double* my_norm, const int* my_bad);
    fy_adam_hparams chunk_hp(const fy_adam_hparams& hp);
    void step_resident(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm);
    void step_streamed(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm);
    void gather_chunk(std::uint32_t c, cudaStream_t s);
    std::uint16_t* chunk_params(std::uint32_t c, int peer) const;

    fy_shard_config cfg_{};
    std::vector<Slice> slices_;
    int pbytes_ = 2, gbytes_ = 2;
    std::uint64_t arena_bytes_ = 0;
    unsigned char* arena_ = nullptr;
    std::vector<unsigned char*> peers_;     // arena base of every rank (own = arena_)
    std::vector<void*> opened_;             // IPC mappings to close
    bool connected_ = false;
    ncclComm_t comm_ = nullptr;
    cudaStream_t opt_ = nullptr, comm_s_ = nullptr;
    cudaEvent_t start_ = nullptr, done_ = nullptr, upd_all_ = nullptr;
    std::vector<cudaEvent_t> chunk_ev_;
    std::vector<cudaEvent_t> upd_t0_;      // timed: after a chunk's grad_ready wait (resident)
    std::vector<char> t0_recorded_;        // upd_t0_[c] recorded this step
    cudaEvent_t upd_start_ = nullptr;      // timed: the resident step's first chunk may start
    std::vector<std::uint32_t> unit_chunk_;      // streamed: the chunk of every pipeline unit
    std::unique_ptr<ChunkPipeline> pipe_;
    std::vector<fy_chunk> units_;
    std::vector<fy_adam_hparams> unit_hp_;
    float* workspace_ = nullptr;
    double* d_norm_ = nullptr;      // this rank's sum of squares
    double* d_total_ = nullptr;     // global sum (after the exchange)
    int* d_nonfinite_ = nullptr;
    int* d_err_ = nullptr;          // barrier timeout flag
    double* h_total_ = nullptr;
    int* h_flags_ = nullptr;        // [nonfinite, barrier error]
    StepCounter counter_{};
    unsigned long long seq_ = 0;
    bool pending_ = false, want_norm_ = false;
    double last_step_ms_ = 0.0;
    std::uint64_t gather_bytes_ = 0, h2d_bytes_ = 0, d2h_bytes_ = 0;
};

// ncclGetUniqueId (rank 0 of a group; the bytes travel out of band)
void nccl_unique_id(void* out);

} // namespace fy
