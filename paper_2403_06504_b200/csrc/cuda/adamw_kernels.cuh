// Internal interface of the fused Adam kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace fy {

// Per-launch scalars, precomputed on the host exactly as DeepSpeed 0.9.3
// cpu_adam.h update_state() does (see adamw_kernels.cu).
struct AdamScalars {
    float beta1, beta2;
    float one_minus_beta1, one_minus_beta2;
    float bias_correction2; // 1 / sqrt(1 - beta2^t)
    float step_size;        // -lr / (1 - beta1^t)
    float w_decay;          // -lr*wd (adamw) or wd (L2 mode)
    float eps;
    float grad_scale;
    int adamw_mode;
    int has_weight_decay;
    // Optional device-side controls, read once per thread at kernel start
    // (enqueue-only clipping / overflow skip, no host sync):
    const float* scale_dev; // effective grad scale = fl(grad_scale * *scale_dev)
    const int* skip_dev;    // *skip_dev != 0: the launch writes nothing
};

// beta^t = float(pow(double(beta), step)) (DeepSpeed's value after a step
// jump or on a fresh optimizer) ...
AdamScalars make_scalars(float lr, float beta1, float beta2, float eps, float weight_decay,
                         std::uint64_t step, int adamw_mode, int bias_correction,
                         float grad_scale);
// ... or given explicitly (b1t / b2t from a StepCounter).
AdamScalars make_scalars_bt(float lr, float beta1, float beta2, float eps, float weight_decay,
                            float b1t, float b2t, int adamw_mode, int bias_correction,
                            float grad_scale);
// Same per-element arithmetic (device-side controls included)?
bool same_scalars(const AdamScalars& a, const AdamScalars& b);

// DeepSpeed 0.9.3 Adam_Optimizer step bookkeeping (csrc/includes/cpu_adam.h
// IncrementStep, called once per adam_update, i.e. once per parameter
// chunk): while the betas are unchanged and the step number advances by one
// per call, beta^t is a float running product (beta_t *= beta); any other
// step number re-evaluates float(pow(double(beta), step)). With K chunks per
// optimizer step, chunk 0 of step t takes the running product
// fl(beta^(t-1) * beta) and chunks 1..K-1 (same step number, so the counter
// "jumps") take pow. A fresh optimizer has step 0 and beta^0 = 1.
struct StepCounter {
    std::uint64_t step = 0;
    float beta1 = 0.0f, beta2 = 0.0f;
    float beta1_t = 1.0f, beta2_t = 1.0f;
    bool constructed = false;  // betas of the constructor (first call's when lazily built)
    void construct(float b1, float b2) {
        beta1 = b1;
        beta2 = b2;
        step = 0;
        beta1_t = beta2_t = 1.0f;
        constructed = true;
    }
    void increment(std::uint64_t t, float b1, float b2);
};

// Fused all-gather epilogue: the updated 16-bit params of this launch are
// also stored at ptr[r] (r < count), each pointing where this rank's slice
// starts inside rank r's full-param buffer — peer (NVLink) pointers on a
// multi-GPU node, local buffers in single-GPU tests.
constexpr int kMaxPeers = 8;
struct Peers {
    void* ptr[kMaxPeers];
    int count;
};

struct AdamLaunch {
    float* master;
    float* m;
    float* v;
    const void* grad;
    int grad_dtype;   // 0 bf16, 1 fp16, 2 fp32
    void* param;      // may be null or alias grad
    int param_dtype;  // 0 bf16, 1 fp16
    std::uint64_t n;
    AdamScalars s;
    double* grad_sq_sum; // optional
    int accumulate_sq;
    float* workspace;    // >= kWorkspaceFloats when grad_sq_sum
    int* nonfinite;      // optional
    Peers peers;         // optional fused gather (count 0 = off)
};

constexpr int kThreads = 256;
constexpr int kMaxChunksPerLaunch = 96;  // multi-chunk launch (the 175B model has 96 blocks)
constexpr std::uint32_t kWorkspaceFloats = 148u * 32u;

// Enqueue the fused step on `stream`. Returns the CUDA launch error.
cudaError_t launch_adamw(const AdamLaunch& a, cudaStream_t stream);

// Loads every kernel of the modules that contain `anchors` (plus this
// file's update kernels) on the CURRENT device. Under CUDA lazy loading
// (the CUDA 12 default) a kernel's first launch loads it, and loading may
// wait for the device to go idle — behind a device barrier that spins until
// a peer's kernel runs, that first launch deadlocks (fy_shard: W shards in
// one fresh process). Idempotent; cheap after the first call per device.
cudaError_t preload_kernels(const void* const* anchors, int count);
// The same step for a list of chunks in ONE persistent TMA launch per
// kMaxChunksPerLaunch chunks (concatenated tile space; grad_sq_sum = the sum
// over the list, taken from list[0] like dtypes, scalars and outputs). Falls
// back to per-chunk launches when the TMA path does not apply.
cudaError_t launch_adamw_multi(const AdamLaunch* list, int count, cudaStream_t stream);

cudaError_t launch_grad_stats(const void* grad, int grad_dtype, std::uint64_t n, float grad_scale,
                              double* grad_sq_sum, int accumulate, float* workspace,
                              int* nonfinite, cudaStream_t stream);

// Global-norm clipping coefficient and overflow flag on the device, from a
// step's accumulated grad sum of squares (of grads already multiplied by the
// stats pass's grad_scale): norm = sqrt(*grad_sq_sum); *scale_out = 1 when
// max_norm <= 0 or norm <= max_norm, else max_norm / (norm + 1e-6) (torch
// clip_grad_norm_); *skip_out = (nonfinite && *nonfinite) or norm not finite.
cudaError_t launch_clip_coef(const double* grad_sq_sum, const int* nonfinite, float max_norm,
                             float* scale_out, int* skip_out, cudaStream_t stream);

// Grid geometry used for the device (cached per device).
struct Geometry {
    int sm_count = 0;
    int ctas_per_sm = 0;
};
Geometry geometry(int device);

// Kernel selection (fy_adamw_tune): path 0 = LSU vector kernel with
// `unroll` quads per thread (1, 2, 4, 8; 0 = 4) and `ctas_per_sm` resident
// CTAs (0 = occupancy limit); path 1 = TMA bulk kernel with `unroll`
// pipeline stages (3, 4, 6; 0 = auto) and `ctas_per_sm` consumer warps (8,
// 16; 0 = auto: 8 on the whole GPU, 16 under an SM budget).
void set_tuning(int path, int unroll, int ctas_per_sm);
// SM budget of the TMA path: at most max_ctas CTAs (one per SM; 0 = all SMs)
// so a concurrent backward keeps the remaining SMs.
void set_max_ctas(int max_ctas);
// Stages / consumer warps the TMA path runs on a device with `sms` SMs under
// the current budget / tuning.
int tma_stages(int sms);
int tma_consumer_warps(int sms, bool fp32_grads = false);
// SM budget of 48..112 CTAs with the automatic shape: 16-bit-gradient launches
// run separate load / store DMA warps and 6 stages.
bool budgeted_split(int sms);
#ifdef FY_SWEEP_VARIANTS
// Sweep build only (build/sweep): TMA variants for bf16 -> bf16: elements
// per stage (1024 | 2048 | 4096), separate load / store DMA warps; probe
// (3 stages x 2048): 1 = L2 evict_first hints, 2 = no arithmetic (the access
// pattern's speed of light; NOT an optimizer), 3 = both, 4-6 DMA orders.
void set_bulk_variant(int tile, int split, int probe);
#endif

// NUMA-local pinned host memory (host_mem.cu). device_numa_node: the GPU's
// node from PCI sysfs (-1 unknown). host_alloc: page-locked, portable,
// preferring `node` (-1: no policy); nullptr on failure; *placed = node of
// the first page when a policy was applied, else -1. host_free: false if p
// did not come from host_alloc. host_numa_node: node of p's page (<0 if
// unknown / unpopulated).
int device_numa_node(int device);
void* host_alloc(std::uint64_t bytes, int node, int* placed);
bool host_free(void* p);
int host_numa_node(const void* p);

} // namespace fy
