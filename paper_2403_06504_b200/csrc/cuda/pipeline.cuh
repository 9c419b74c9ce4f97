// Chunk pipeline for the streamed (out-of-core) optimizer step.
#pragma once

#include "adamw_kernels.cuh"
#include "fuyou/fy_adam.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace fy {

// Raised for CUDA failures; the C ABI maps it to FY_ERR_DEVICE.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char* what);

// Kernel scalars of one update: beta^t from hp (given) or pow(step).
AdamScalars scalars_of(const fy_adam_hparams& hp);
// fy_adam_counter <-> StepCounter
StepCounter load_counter(const fy_adam_counter& c);
void store_counter(const StepCounter& k, fy_adam_counter* c);

// Device staging for one chunk in flight: [master | m | v] (12n B), plus a
// gradient area (host-sourced grads) and a param area (downcast output).
struct Slot {
    unsigned char* states = nullptr;
    void* grad = nullptr;
    void* param = nullptr;
};

class ChunkPipeline {
public:
    explicit ChunkPipeline(const fy_pipeline_config& cfg);
    ~ChunkPipeline();
    void release() noexcept;  // frees everything allocated so far (dtor, failed ctor)
    ChunkPipeline(const ChunkPipeline&) = delete;
    ChunkPipeline& operator=(const ChunkPipeline&) = delete;

    // per_chunk_hp (optional, count entries): each unit's own hyper-parameters
    // (the sharded step passes one chunk's beta^t to all of its pieces);
    // start_after (optional): the step's first operations wait on this event.
    void step(const fy_chunk* chunks, std::uint32_t count, const fy_adam_hparams& hp,
              bool want_norm, const fy_adam_hparams* per_chunk_hp = nullptr,
              cudaEvent_t start_after = nullptr);
    void wait(double* grad_sq_sum, int* nonfinite);
    void timings(fy_chunk_timing* out, std::uint32_t count, std::uint64_t* step_ns) const;
    // device-side clip coefficient / overflow-skip flag for the following
    // steps (fy_clip_coef outputs; nullptr = off)
    void set_controls(const float* scale_dev, const int* skip_dev) {
        scale_dev_ = scale_dev;
        skip_dev_ = skip_dev;
    }

    cudaStream_t h2d_stream() const { return h2d_; }
    cudaStream_t d2h_stream() const { return d2h_; }
    cudaStream_t compute_stream() const { return opt_; }
    // device-side sum of squares / non-finite flag of the step in flight and
    // the event recorded when all of its work (copies included) is done
    double* device_norm() const { return d_norm_; }
    int* device_nonfinite() const { return d_nonfinite_; }
    cudaEvent_t step_end_event() const { return step_end_; }
    // the step's work is complete (host side: marks it waited without a sync)
    void mark_waited() { pending_ = false; }

private:
    enum Ev { kH2dStart, kH2dEnd, kUpdStart, kUpdEnd, kD2hStart, kD2hEnd, kEvPerChunk };
    cudaEvent_t ev(std::uint32_t chunk, int which) const { return events_[chunk * kEvPerChunk + which]; }
    void ensure_events(std::uint32_t count);
    // states of this chunk live in device memory (the whole pipeline's
    // states_on_device, or the chunk's FY_CHUNK_STATES_ON_DEVICE flag)
    bool resident(const fy_chunk& c) const {
        return cfg_.states_on_device || (c.flags & FY_CHUNK_STATES_ON_DEVICE) != 0;
    }
    void issue_h2d(std::uint32_t i);
    void issue_update(std::uint32_t i);
    void issue_d2h(std::uint32_t i);

    fy_pipeline_config cfg_{};
    int grad_bytes_ = 2;
    int param_bytes_ = 2;
    cudaStream_t h2d_ = nullptr, d2h_ = nullptr, opt_ = nullptr;
    std::vector<Slot> slots_;
    std::vector<cudaEvent_t> events_;
    cudaEvent_t step_start_ = nullptr;
    cudaEvent_t step_end_ = nullptr;
    float* workspace_ = nullptr;
    double* d_norm_ = nullptr;
    int* d_nonfinite_ = nullptr;
    double* h_norm_ = nullptr;
    int* h_nonfinite_ = nullptr;
    bool want_norm_ = false;
    bool pending_ = false;
    bool have_prev_ = false;
    std::uint32_t last_count_ = 0;
    // Current step's inputs (valid during step()).
    const fy_chunk* chunks_ = nullptr;
    fy_adam_hparams hp_{};
    const fy_adam_hparams* unit_hp_ = nullptr;
    StepCounter counter_{};  // DeepSpeed Adam_Optimizer step bookkeeping (unless no_step_counter)
    const float* scale_dev_ = nullptr;
    const int* skip_dev_ = nullptr;
};

} // namespace fy
