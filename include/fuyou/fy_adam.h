/* fy_adam.h — C ABI of the B200 out-of-core Adam step (kernels + chunk
 * pipeline). Plain pointers and sizes only; no CUDA, torch or C++ types.
 * `stream` arguments are cudaStream_t values passed as void* (NULL = the
 * legacy default stream).
 *
 * Conventions follow the reference C ABI (proj/include/offsim/offsim_c.h:
 * 16-28, proj/src/capi.cpp:19-51): integer status codes with the same
 * numbering, a thread-local last-error string that is never NULL, no
 * exception crossing the boundary, NULL arguments -> FY_ERR_CONFIG. The
 * caller owns every buffer; nothing here allocates device memory except the
 * pipeline object (its staging slots), which fy_pipeline_destroy releases.
 *
 * Reference interfaces replaced (the reference prices these as DAG tasks;
 * this library executes them):
 *   fy_adamw_chunk       <- `opt update gK`, TaskKind::optimizer_update on
 *                           ResourceId::cpu_compute, work = 12h^2 params
 *                           (proj/src/task_graph.cpp:488-495; priced at
 *                           proj/src/simulator.cpp:21,37-41)
 *   fy_pipeline_step     <- the optimizer group block `opt state_s2c gK ->
 *                           opt update gK -> opt state_c2s gK / opt
 *                           param_c2s gK` with the depth-2 read gate
 *                           (proj/src/task_graph.cpp:453-503)
 *   fy_swap_out / _in    <- activation swap transfers `fwd act_g2c/act_c2s`,
 *                           `fwd ckpt_g2c/ckpt_c2s`, `bwd ckpt_s2c/ckpt_c2g`,
 *                           `bwd act_s2c/act_c2g`
 *                           (proj/src/task_graph.cpp:296-321,357-397)
 */
#ifndef FUYOU_FY_ADAM_H
#define FUYOU_FY_ADAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fy_status {
    FY_OK = 0,
    FY_ERR_CONFIG = 2,     /* bad argument / unsupported combination   */
    FY_ERR_INFEASIBLE = 3, /* does not fit (device or host memory)     */
    FY_ERR_INVARIANT = 4,  /* executed trace violates its graph        */
    FY_ERR_INTERNAL = 5,
    FY_ERR_DEVICE = 6      /* CUDA / NCCL / IO error (message in last error) */
} fy_status;

typedef enum fy_dtype { FY_BF16 = 0, FY_FP16 = 1, FY_FP32 = 2 } fy_dtype;

const char* fy_version(void);
const char* fy_last_error(void);

/* Adam hyper-parameters of one step. Semantics: DeepSpeed 0.9.3
 * DeepSpeedCPUAdam (the optimizer the paper runs),
 * csrc/includes/cpu_adam.h update_state: bias_correction1 = 1 - beta1^t,
 * bias_correction2 = 1 / sqrtf(1 - beta2^t) (float ops), eps added after the
 * bias-corrected sqrt(v), decoupled decay when adamw_mode != 0. The gradient
 * is first multiplied by grad_scale (1/loss_scale, times a clip coefficient
 * if the caller clips).
 * beta^t: beta_t_given == 0 -> float(pow(double(beta), step)), the value a
 * fresh DeepSpeed optimizer or a step-number jump produces; beta_t_given != 0
 * -> beta1_t / beta2_t as given, e.g. by fy_adam_counter_next, which keeps
 * DeepSpeed's running product across consecutive calls. */
typedef struct fy_adam_hparams {
    float lr;
    float beta1;
    float beta2;
    float eps;
    float weight_decay;
    uint64_t step; /* 1-based step count after this update */
    int adamw_mode;
    int bias_correction;
    float grad_scale;
    int beta_t_given;
    float beta1_t;
    float beta2_t;
} fy_adam_hparams;

/* DeepSpeed's per-optimizer step bookkeeping (cpu_adam.h Adam_Optimizer::
 * IncrementStep, run once per adam_update call = once per parameter chunk):
 * with unchanged betas and a step number one past the counter's, beta^t is
 * the float running product beta_t *= beta; otherwise (first call of a step
 * whose chunk 0 already advanced the counter, a restart, changed betas)
 * beta^t = float(pow(double(beta), step)). So in a step over K chunks, chunk
 * 0 takes fl(beta^(t-1) * beta) and chunks 1..K-1 take pow — bit for bit
 * what DeepSpeedCPUAdam hands its kernel. init = the optimizer's constructor
 * (step 0, beta^0 = 1). next: IncrementStep(hp->step, hp->beta1, hp->beta2),
 * then writes hp->beta1_t / beta2_t and sets hp->beta_t_given. */
typedef struct fy_adam_counter {
    uint64_t step;
    float beta1, beta2;
    float beta1_t, beta2_t;
    int constructed; /* 0: constructed lazily with the first call's betas */
} fy_adam_counter;
fy_status fy_adam_counter_init(fy_adam_counter* c, float beta1, float beta2);
fy_status fy_adam_counter_next(fy_adam_counter* c, fy_adam_hparams* hp);

/* One chunk (one transformer block = 12h^2 params, or a shard slice of it).
 * master / exp_avg / exp_avg_sq: fp32 [n] device pointers, updated in place.
 * grad: [n] of grad_dtype (bf16/fp16/fp32), device.
 * param_out: [n] of param_dtype (bf16/fp16) or NULL; may alias grad (the
 * reference's "gradient buffer becomes the fp16 params",
 * task_graph.cpp:493-495).
 * grad_sq_sum: optional device double; receives sum((grad*grad_scale)^2)
 * (added to the existing value when accumulate_sq != 0). Requires workspace.
 * workspace: device floats, >= fy_adamw_workspace_floats() (may be NULL when
 * grad_sq_sum is NULL).
 * nonfinite_flag: optional device int, set to 1 if any scaled gradient is
 * inf/nan (never cleared by the kernel). */
typedef struct fy_adamw_args {
    float* master;
    float* exp_avg;
    float* exp_avg_sq;
    const void* grad;
    int grad_dtype;
    void* param_out;
    int param_dtype;
    uint64_t n;
    fy_adam_hparams hp;
    double* grad_sq_sum;
    int accumulate_sq;
    float* workspace;
    int* nonfinite_flag;
    /* Optional device-side controls (enqueue-only clipping / overflow skip;
     * see fy_clip_coef). NULL = off. */
    const float* grad_scale_dev; /* effective scale = fl(hp.grad_scale * *grad_scale_dev) */
    const int* skip_if_set;      /* *skip_if_set != 0: states untouched, params
                                    rewritten from the unchanged master (the
                                    param buffer may alias this step's grads) */
} fy_adamw_args;

uint32_t fy_adamw_workspace_floats(void);

/* Fused unscale + grad-norm partial + AdamW + downcast, one launch (two when
 * grad_sq_sum is requested: the second is a one-block ordered reduction).
 * n == 0, or a launch skipped by *skip_if_set, contributes 0 to grad_sq_sum
 * (written as 0 when accumulate_sq == 0). */
fy_status fy_adamw_chunk(const fy_adamw_args* args, void* stream);

/* The same step for `count` chunks at once (multi-tensor apply): one
 * persistent TMA launch covers up to 96 chunks (their tiles concatenated),
 * so a step over many small blocks pays one ramp-up / drain / tail instead
 * of one per chunk (chunks of >= 33.5M elements, where that overhead is
 * under 2%, keep their own launch). Entries may differ in hp (runs of equal
 * hyper-parameters share a launch: DeepSpeed's counter gives chunk 0 of a
 * step its own beta^t) but must share dtypes, param_out presence, the
 * device-side controls and the statistics outputs (grad_sq_sum,
 * accumulate_sq, workspace, nonfinite_flag); grad_sq_sum receives the sum
 * over all chunks. Results
 * per element are identical to count fy_adamw_chunk calls (the grad sum of
 * squares up to summation order). Chunks must not overlap. */
fy_status fy_adamw_chunks(const fy_adamw_args* list, uint32_t count, void* stream);

/* Same step with the all-gather fused into the epilogue:
 * besides param_out (required: the local copy), every updated 16-bit param
 * is stored to dst[r] (r < ndst <= 8), where dst[r] points at the start of
 * THIS rank's slice inside rank r's full-param buffer — peer pointers
 * (NVLink, e.g. IPC / symmetric memory) on a multi-GPU node. Replaces the
 * separate ncclAllGather of the updated bf16 slices; the caller orders the
 * peers' reads after this launch (event / barrier). */
fy_status fy_adamw_chunk_gather(const fy_adamw_args* args, void* const* dst, uint32_t ndst,
                                void* stream);

/* Gradient statistics only (2 B/param read): sum of squares and non-finite
 * flag, for callers that must clip or skip before any update is applied. */
fy_status fy_grad_stats(const void* grad, int grad_dtype, uint64_t n, float grad_scale,
                        double* grad_sq_sum, int accumulate_sq, float* workspace,
                        int* nonfinite_flag, void* stream);

/* Global-norm clipping and fp16-overflow skip without a host round trip
 * (the DeepSpeed engine clips / skips before its CPU Adam step): after a
 * stats pass over every chunk (fy_grad_stats with the loss-scale inverse,
 * accumulating into *grad_sq_sum and *nonfinite), one 1-thread kernel
 * writes *scale_out = 1, or max_norm / (norm + 1e-6) when max_norm > 0 and
 * norm = sqrt(*grad_sq_sum) exceeds it (torch clip_grad_norm_), and
 * *skip_out = 1 when any gradient was non-finite. Pass scale_out as
 * grad_scale_dev and skip_out as skip_if_set to the fy_adamw_chunk(s)
 * launches of the step (with hp.grad_scale = the loss-scale inverse). All
 * pointers are device memory; stream-ordered. */
fy_status fy_clip_coef(const double* grad_sq_sum, const int* nonfinite, float max_norm,
                       float* scale_out, int* skip_out, void* stream);

/* Kernel selection of the fused step (every choice computes the same bits),
 * process-wide.
 * path 0: LSU kernel, `unroll` quads (4 elements) per thread per grid-stride
 *         iteration in {1,2,4,8} (0 = 4), `ctas_per_sm` resident CTAs
 *         (0 = occupancy);
 * path 1: TMA bulk-copy kernel (cp.async.bulk + mbarrier, one CTA of 8 or
 *         16 consumer warps + 1 DMA warp per SM), `unroll` = pipeline stages
 *         in {3,4,6} (fp32 grads: 3 or 6; 0 = auto: 3 on the whole GPU, 4
 *         under an SM budget), third argument = consumer warps {8,16}
 *         (0 = auto: 8 on the whole GPU, 16 under an SM budget).
 * Default: path 1, auto (measured best, profiles/). */
fy_status fy_adamw_tune(int path, int unroll, int ctas_per_sm);
/* SM budget of the fused step (TMA path), process-wide: launches use at most
 * max_ctas CTAs — one per SM — leaving the other SMs to a backward running
 * concurrently on another stream (0 = every SM, the default). Budgeted
 * launches run the deeper pipeline (more bytes in flight per SM). */
fy_status fy_adamw_sm_budget(int max_ctas);

/* Number of SMs and the launch geometry the kernels use on `device`
 * (diagnostics / roofline bookkeeping). */
fy_status fy_device_info(int device, int* sm_count, int* ctas_per_sm, int* threads_per_cta);

/* ------------------------------------------------------------------ */
/* Multi-GPU sharding of a chunk: chunk of n elements split
 * into `world` contiguous slices, each a multiple of `align` elements except
 * the last; returns [offset, count) of `rank`. Pure host arithmetic. */
fy_status fy_shard_range(uint64_t n, uint32_t world, uint32_t rank, uint32_t align,
                         uint64_t* offset, uint64_t* count);

/* ------------------------------------------------------------------ */
/* Sharded optimizer step across the GPUs of one node (the
 * reference's single-GPU optimizer group block, proj/src/task_graph.cpp:
 * 453-503, with every block split by parameter slice). One fy_shard per GPU
 * (one process per GPU, or one per device in a single process). Rank r owns
 * slice r (fy_shard_range, 8-element aligned) of every chunk: the caller
 * hands it that slice's fp32 [master|m|v] (device memory for
 * FY_TIER_DEVICE; pinned host memory, ideally fy_host_alloc'd NUMA-local,
 * for FY_TIER_HOST, streamed through a chunk pipeline) and the slice's
 * gradients (device). A step updates every owned slice with the fused kernel
 * and all-gathers the updated 16-bit params, so that every rank ends the
 * step holding every chunk's full params in the shard's ARENA (device memory
 * owned by the shard; fy_shard_slice_info gives each chunk's pointer).
 *
 * Gather (world > 1):
 *   FY_GATHER_NCCL  ncclAllGather, in place, per chunk on a comm stream, as
 *                   soon as the chunk's slice is updated (overlaps the next
 *                   chunks). Needs nccl_id (fy_nccl_unique_id on rank 0,
 *                   broadcast out of band).
 *   FY_GATHER_PEER  no collective: the update kernel's epilogue stores every
 *                   param into every peer's arena through NVLink (resident
 *                   tier; the streamed tier pushes each slice with the copy
 *                   engines), ordered by device-side barriers at the start
 *                   and end of the step. The peers' arenas come from
 *                   fy_shard_ipc_handle + fy_shard_connect (processes),
 *                   fy_shard_connect_ptrs (one process), or — when nccl_id
 *                   is given — an NCCL all-gather of the handles at create.
 * The PEER barriers need every rank's stream to make progress while another
 * rank's barrier spins: one process per GPU always has that; a process that
 * drives several shards on ONE device must keep its streams (3 per shard)
 * within CUDA_DEVICE_MAX_CONNECTIONS (default 8; streams beyond it share
 * hardware queues and serialise: 8 shards on one device need 32). Every
 * kernel a step may launch is loaded at fy_shard_create (under CUDA's lazy
 * loading a first launch behind a spinning barrier would deadlock). A
 * barrier that waits > 120 s (env FY_BARRIER_TIMEOUT_S) gives up and
 * fy_shard_wait reports FY_ERR_DEVICE instead of hanging the GPU.
 * In-place gradients: io.grad may point at this rank's own slot of the
 * chunk's arena region (fy_shard_slice.params + rank * stride elements,
 * 16-bit grads): the update then overwrites the gradients with the params,
 * the reference's convention (proj/src/task_graph.cpp:493-495), and the
 * caller needs no separate gradient memory.
 * want_grad_norm: the GLOBAL sum of squares over all ranks (one 8-byte
 * all-reduce, or the exit barrier's exchange summed in rank order).
 * Step counter: one DeepSpeed IncrementStep per chunk (fy_adam_counter
 * semantics) unless no_step_counter or hp->beta_t_given. */
enum { FY_GATHER_NONE = 0, FY_GATHER_NCCL = 1, FY_GATHER_PEER = 2 };
enum { FY_TIER_DEVICE = 0, FY_TIER_HOST = 1 };
#define FY_NCCL_ID_BYTES 128

fy_status fy_nccl_unique_id(void* id_out);

typedef struct fy_shard fy_shard;
typedef struct fy_shard_config {
    int device;
    uint32_t world, rank;
    int gather;                  /* FY_GATHER_*; world 1: none                 */
    const void* nccl_id;         /* FY_NCCL_ID_BYTES or NULL                   */
    int tier;                    /* FY_TIER_DEVICE | FY_TIER_HOST              */
    uint32_t chunk_count;
    const uint64_t* chunk_elems; /* full chunk sizes, identical on every rank  */
    int grad_dtype;
    int param_dtype;
    uint32_t slots;              /* FY_TIER_HOST: staging slots (0 = 3)        */
    uint64_t piece_elems;        /* FY_TIER_HOST: max elements per pipeline
                                    unit (0 = a whole slice)                   */
    int params_to_host;          /* also D2H each updated slice to io.h_param  */
    int no_step_counter;
    int grads_on_host;           /* io.grad is pinned HOST memory: each slice's
                                    grads go H2D through the chunk pipeline
                                    (with FY_TIER_DEVICE the states stay in
                                    HBM; io.grad and io.h_param may alias)   */
} fy_shard_config;

typedef struct fy_shard_slice {
    uint64_t offset, count;      /* this rank's slice of the chunk             */
    uint64_t stride;             /* padded slice length of every rank          */
    void* params;                /* device: the chunk's full params (arena)    */
} fy_shard_slice;

typedef struct fy_shard_io {     /* one per chunk: this rank's buffers         */
    void* states;                /* [master|m|v] of the slice, 12*count bytes  */
    const void* grad;            /* [count] gradients of the slice: device, or
                                    pinned host with grads_on_host           */
    void* h_param;               /* pinned host [count] (params_to_host)       */
    void* grad_ready;            /* optional cudaEvent_t                       */
} fy_shard_io;

typedef struct fy_shard_stats {
    double step_ms;              /* last step, device time (events)            */
    uint64_t gather_bytes;       /* param bytes this rank sent to peers        */
    uint64_t h2d_bytes, d2h_bytes;
    uint32_t world, rank;
    int gather;                  /* effective FY_GATHER_*                      */
    int stages;                  /* TMA pipeline stages of the update kernel   */
    int consumer_warps;          /* TMA consumer warps per CTA                 */
} fy_shard_stats;

fy_status fy_shard_create(const fy_shard_config* cfg, fy_shard** out);
void fy_shard_destroy(fy_shard* s);
fy_status fy_shard_slice_info(const fy_shard* s, uint32_t chunk, fy_shard_slice* out);
/* The arena: device base pointer and size (header + every chunk's params). */
fy_status fy_shard_arena(const fy_shard* s, void** base, uint64_t* bytes);
fy_status fy_shard_ipc_handle(const fy_shard* s, void* handle_out);
fy_status fy_shard_connect(fy_shard* s, const void* handles);
fy_status fy_shard_connect_ptrs(fy_shard* s, void* const* arenas);
/* Enqueues one optimizer step after the work already on `stream` and makes
 * `stream` wait for its completion (gather included); returns without
 * blocking. fy_shard_wait blocks until it is done. */
fy_status fy_shard_step(fy_shard* s, const fy_shard_io* io, const fy_adam_hparams* hp,
                        int want_grad_norm, void* stream);
fy_status fy_shard_wait(fy_shard* s, double* grad_sq_sum, int* nonfinite);
fy_status fy_shard_get_stats(const fy_shard* s, fy_shard_stats* out);
/* Device time of each chunk's update kernel(s) in the last waited step, ms
 * (resident: one event per chunk on the shard's update stream, the chunk's
 * fused update + norm reduction from the previous chunk's end, the step's
 * start or its grad_ready; streamed tier: the sum over the chunk's pipeline
 * pieces' update kernels). */
fy_status fy_shard_update_ms(const fy_shard* s, double* chunk_ms, uint32_t count);

/* ------------------------------------------------------------------ */
/* Chunk pipeline: streamed (out-of-core) optimizer step.
 *
 * The host holds each chunk's states as one contiguous pinned region
 * [master | exp_avg | exp_avg_sq] (12n bytes) and optionally its gradients
 * and output params. Per chunk the pipeline issues:
 *   H2D states (copy stream)  -> fy_adamw_chunk (compute stream)
 *   -> D2H states (+ params)  (copy stream)
 * with `slots` device staging buffers, and the reference's depth-2 read gate
 * (the read of chunk i waits for the update of chunk i-2,
 * task_graph.cpp:463-471). Gradients may live on the device (produced by
 * backward; optionally gated by a caller event) or on the host (H2D'd with
 * the states). */

typedef struct fy_pipeline fy_pipeline;

typedef struct fy_pipeline_config {
    int device;
    uint64_t max_chunk_elems;   /* largest chunk; sizes the staging slots */
    uint32_t slots;             /* device staging slots (>= 2; default 3) */
    int grad_dtype;
    int param_dtype;
    int grads_on_host;          /* 1: grads come from pinned host memory  */
    int params_to_host;         /* 1: D2H the downcast params to host     */
    int keep_params_on_device;  /* 1: also write params to chunk.d_param  */
    int states_on_device;       /* 1: chunk.h_states is a DEVICE pointer to
                                   [master|m|v]; no state copies (the
                                   device-resident tier; grads/params may
                                   still cross the host link) */
    int no_step_counter;        /* 0 (default): the pipeline is the optimizer
                                   object and keeps DeepSpeed's step counter
                                   (fy_adam_counter semantics, one increment
                                   per chunk update) unless hp->beta_t_given;
                                   1: every chunk uses hp as given */
} fy_pipeline_config;

typedef struct fy_chunk {
    uint64_t n;
    void* h_states;       /* [master|m|v], 12n bytes: pinned host, or device
                             when states_on_device (required)              */
    const void* grad;     /* device ptr (grads_on_host=0) or pinned host ptr */
    void* h_param;        /* pinned host [n] params (params_to_host=1)      */
    void* d_param;        /* device [n] params (keep_params_on_device=1)    */
    void* grad_ready;     /* optional cudaEvent_t the update must wait on   */
    uint64_t states_stride; /* elements from master to m and m to v in
                               h_states (0 = n, i.e. contiguous [master|m|v]);
                               > n lets a piece of a larger chunk's SoA
                               arrays be one pipeline unit               */
    void* update_done;    /* optional cudaEvent_t recorded right after this
                             chunk's update (e.g. to start its all-gather
                             on another stream while the next chunks are
                             still streaming)                            */
    uint32_t flags;       /* FY_CHUNK_STATES_ON_DEVICE: this chunk's
                             h_states is DEVICE memory kept resident in HBM
                             (no state copies; params still go to h_param) —
                             lets spare HBM hold part of an out-of-core
                             model's optimizer states                   */
} fy_chunk;
#define FY_CHUNK_STATES_ON_DEVICE 1u

/* Per-chunk timings of the last step, in ns relative to the step start
 * (CUDA events): h2d [start,end), update [start,end), d2h [start,end). */
typedef struct fy_chunk_timing {
    uint64_t h2d_start_ns, h2d_end_ns;
    uint64_t upd_start_ns, upd_end_ns;
    uint64_t d2h_start_ns, d2h_end_ns;
} fy_chunk_timing;

fy_status fy_pipeline_create(const fy_pipeline_config* cfg, fy_pipeline** out);
void fy_pipeline_destroy(fy_pipeline* p);

/* Runs one optimizer step over chunks[0..count) in the given order and
 * returns when the step has been ENQUEUED; fy_pipeline_wait blocks until it
 * completes. grad_sq_sum (optional, host double*) receives the step's sum of
 * squared scaled gradients after fy_pipeline_wait. */
fy_status fy_pipeline_step(fy_pipeline* p, const fy_chunk* chunks, uint32_t count,
                           const fy_adam_hparams* hp, int want_grad_norm);
fy_status fy_pipeline_wait(fy_pipeline* p, double* grad_sq_sum, int* nonfinite);

/* Device-side clip coefficient / overflow-skip flag (fy_clip_coef outputs)
 * applied by the following steps' updates (NULL = off). A skipped update
 * leaves the states unchanged and still writes the params (from the
 * unchanged master), so the write-backs stay correct. */
fy_status fy_pipeline_set_controls(fy_pipeline* p, const float* grad_scale_dev, const int* skip_if_set);

/* Timings of the last completed step (count entries). */
fy_status fy_pipeline_timings(const fy_pipeline* p, fy_chunk_timing* out, uint32_t count,
                              uint64_t* step_ns);

/* ------------------------------------------------------------------ */
/* Whole-iteration execution of a scenario's task graph on the GPU with
 * caller-owned optimizer states (one fy_chunk per transformer block, n =
 * 12h^2; h_states pinned host [master|m|v], h_param pinned host bf16 output,
 * grad a device bf16 pointer). Same semantics as offsim_execute (see
 * include/offsim/exec.hpp); the summary JSON is library-allocated (free it
 * with offsim_string_free). Errors are reported through offsim_last_error.
 * chunk_count 0 = synthetic states. */
fy_status fy_graph_execute(const char* scenario_json, const char* exec_opts_json,
                           const fy_chunk* chunks, uint32_t chunk_count, char** summary_json_out);

/* ------------------------------------------------------------------ */
/* Activation swap engine: the GPU -> pinned host (-> SSD) copy path of the
 * reference's activation swap tasks (`fwd act_g2c/act_c2s`, `fwd
 * ckpt_g2c/ckpt_c2s`, `bwd ckpt_s2c/ckpt_c2g`, `bwd act_s2c/act_c2g`,
 * proj/src/task_graph.cpp:296-321,357-397), callable by a training
 * framework. placement = the planner's checkpoint location
 * (proj/src/runner.cpp:90-106): FY_SWAP_CPU keeps the bytes in NUMA-local
 * pinned memory, FY_SWAP_SSD streams them through a ring of `slots` pinned
 * buffers of `slot_bytes` into an O_DIRECT file under `file_dir` (io_uring).
 * All calls only ENQUEUE work (two copy streams + an IO stream); ordering
 * with the caller uses CUDA events: `ready` (optional) is waited on before
 * reading the source / writing the destination, `src_free` is recorded when
 * the swapped-out device buffer may be reused, `done` when the swapped-in
 * data is on the device. A swapper is used by one thread at a time. */
typedef struct fy_swapper fy_swapper;
enum { FY_SWAP_CPU = 0, FY_SWAP_SSD = 1 };
typedef struct fy_swap_config {
    int device;
    uint64_t slot_bytes;  /* SSD ring slot size (0: 64 MiB; rounded to 4 KiB) */
    uint32_t slots;       /* ring slots (0: 4; >= 2)                          */
    const char* file_dir; /* NULL: /tmp; "d1:d2:..." = one directory per SSD,
                             the swap file striped RAID-0 over them (4 MiB) */
    int direct_io;        /* O_DIRECT for the swap file                       */
} fy_swap_config;

fy_status fy_swapper_create(const fy_swap_config* cfg, fy_swapper** out);
void fy_swapper_destroy(fy_swapper* s);
fy_status fy_swap_out(fy_swapper* s, const void* dev_src, uint64_t bytes, int placement,
                      void* ready_event, void* src_free_event, uint64_t* handle_out);
fy_status fy_swap_in(fy_swapper* s, uint64_t handle, void* dev_dst, void* ready_event,
                     void* done_event);
/* Frees the handle's host buffer / file region (blocks until its queued
 * copies finished). */
fy_status fy_swap_release(fy_swapper* s, uint64_t handle);
/* Blocks until all queued swaps finished; reports file IO errors. */
fy_status fy_swapper_sync(fy_swapper* s);
/* Pinned host bytes allocated for CPU placement, bytes currently laid out
 * in the swap file, and the IO engine ("io_uring" | "pread/pwrite"). */
fy_status fy_swapper_stats(const fy_swapper* s, uint64_t* host_bytes, uint64_t* file_bytes,
                           const char** io_engine);

/* Peer buffers for the fused all-gather epilogue without torch symmetric
 * memory: fy_ipc_alloc allocates device memory and writes its 64-byte CUDA
 * IPC handle; another process opens it with fy_ipc_open (peer access enabled
 * lazily) and passes the returned pointer (+ its slice offset) as a
 * fy_adamw_chunk_gather destination. Close with fy_ipc_close in the opener,
 * free with fy_ipc_free in the allocator. */
#define FY_IPC_HANDLE_BYTES 64
fy_status fy_ipc_alloc(uint64_t bytes, void** ptr, void* handle_out);
fy_status fy_ipc_open(const void* handle, void** ptr);
fy_status fy_ipc_close(void* ptr);
fy_status fy_ipc_free(void* ptr);

/* Pinned host allocation (page-locked, portable) on the NUMA node of the
 * GPU that will stream it — the host tier's "NUMA-local pinned memory"
 * (SURVEY.md §8e). fy_host_alloc: the current device's node (PCI sysfs).
 * fy_host_alloc_on: numa_node >= 0 prefers that node, -1 the current
 * device's node, -2 no placement policy. Falls back to cudaHostAlloc when
 * registration is refused. Free either with fy_host_free. */
fy_status fy_host_alloc(uint64_t bytes, void** out);
fy_status fy_host_alloc_on(uint64_t bytes, int numa_node, void** out);
fy_status fy_host_free(void* p);
/* NUMA node of a GPU (-1 if the platform does not report one) and of the
 * page holding p (< 0 if unknown). */
fy_status fy_device_numa_node(int device, int* node);
fy_status fy_host_numa_node(const void* p, int* node);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FUYOU_FY_ADAM_H */
