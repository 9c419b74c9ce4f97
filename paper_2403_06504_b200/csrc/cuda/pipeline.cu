// Streamed optimizer step: the executor of the reference's optimizer group
// block (proj/src/task_graph.cpp:453-503) on one B200.
//
//   reference task            here
//   opt state_s2c gK      ->  H2D of [master|m|v] into a staging slot (copy
//                             stream h2d_), from pinned host memory
//   opt update gK         ->  fused AdamW kernel on the compute stream opt_,
//                             after its state read and its gradient
//                             (bwd grad_g2c bK: grads stay in HBM, the
//                             kernel waits on the producer's event instead)
//   opt state_c2s gK      ->  D2H of the updated states (copy stream d2h_)
//   opt param_c2s gK      ->  D2H of the downcast params
//
// Read gate: as in task_graph.cpp:463-471 the read of group m waits for the
// update of group m-2, so at most two groups are read ahead of the update
// pipeline (delayed write-back). Slot reuse adds the physical
// constraint the DES models as a memory pool: the read into a slot waits for
// the write-back of the group that last used it.
//
// Operations are enqueued from one host thread in an order where every event
// a stream waits on has already been recorded (H2D(0); then per i: update(i),
// D2H(i), H2D(i+1)), so the whole step is issued without host blocking and
// the three engines (H2D copy, SMs, D2H copy) overlap.

#include "pipeline.cuh"

#include <cstring>

namespace fy {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                          cudaGetErrorString(e) + ")");
}

AdamScalars scalars_of(const fy_adam_hparams& hp) {
    if (hp.beta_t_given)
        return make_scalars_bt(hp.lr, hp.beta1, hp.beta2, hp.eps, hp.weight_decay, hp.beta1_t, hp.beta2_t,
                               hp.adamw_mode, hp.bias_correction, hp.grad_scale);
    return make_scalars(hp.lr, hp.beta1, hp.beta2, hp.eps, hp.weight_decay, hp.step, hp.adamw_mode,
                        hp.bias_correction, hp.grad_scale);
}

StepCounter load_counter(const fy_adam_counter& c) {
    StepCounter k;
    k.step = c.step;
    k.beta1 = c.beta1;
    k.beta2 = c.beta2;
    k.beta1_t = c.beta1_t;
    k.beta2_t = c.beta2_t;
    k.constructed = c.constructed != 0;
    return k;
}

void store_counter(const StepCounter& k, fy_adam_counter* c) {
    c->step = k.step;
    c->beta1 = k.beta1;
    c->beta2 = k.beta2;
    c->beta1_t = k.beta1_t;
    c->beta2_t = k.beta2_t;
    c->constructed = k.constructed ? 1 : 0;
}

namespace {
int dtype_bytes(int dt) { return dt == FY_FP32 ? 4 : 2; }
} // namespace

ChunkPipeline::ChunkPipeline(const fy_pipeline_config& cfg) : cfg_(cfg) {
    if (cfg_.slots == 0) cfg_.slots = 3;
    if (cfg_.slots < 2) throw ArgError("pipeline: slots must be >= 2");
    if (cfg_.max_chunk_elems == 0) throw ArgError("pipeline: max_chunk_elems must be > 0");
    if (cfg_.grad_dtype < FY_BF16 || cfg_.grad_dtype > FY_FP32)
        throw ArgError("pipeline: bad grad_dtype");
    if (cfg_.param_dtype != FY_BF16 && cfg_.param_dtype != FY_FP16)
        throw ArgError("pipeline: param_dtype must be bf16 or fp16");
    grad_bytes_ = dtype_bytes(cfg_.grad_dtype);
    param_bytes_ = dtype_bytes(cfg_.param_dtype);

    try {
        check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
        int lo = 0, hi = 0;
        check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
        check_cuda(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "h2d stream");
        check_cuda(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "d2h stream");
        // The update kernel is short next to the copies; give it the higher
        // priority so it is not queued behind a synthetic backward.
        check_cuda(cudaStreamCreateWithPriority(&opt_, cudaStreamNonBlocking, hi), "opt stream");

        const std::uint64_t n = cfg_.max_chunk_elems;
        slots_.resize(cfg_.slots);
        for (Slot& s : slots_) {
            if (!cfg_.states_on_device) check_cuda(cudaMalloc(&s.states, 12ull * n), "slot states");
            if (cfg_.grads_on_host) check_cuda(cudaMalloc(&s.grad, grad_bytes_ * n), "slot grad");
            if (cfg_.params_to_host) check_cuda(cudaMalloc(&s.param, param_bytes_ * n), "slot param");
        }
        check_cuda(cudaMalloc(&workspace_, sizeof(float) * kWorkspaceFloats), "workspace");
        check_cuda(cudaMalloc(&d_norm_, sizeof(double)), "norm");
        check_cuda(cudaMalloc(&d_nonfinite_, sizeof(int)), "nonfinite");
        check_cuda(cudaHostAlloc(&h_norm_, sizeof(double), cudaHostAllocDefault), "h norm");
        check_cuda(cudaHostAlloc(&h_nonfinite_, sizeof(int), cudaHostAllocDefault), "h nonfinite");
        check_cuda(cudaEventCreate(&step_start_), "event");
        check_cuda(cudaEventCreate(&step_end_), "event");
    } catch (...) {
        release();  // a failed allocation must not leak the earlier ones
        throw;
    }
}

ChunkPipeline::~ChunkPipeline() { release(); }

void ChunkPipeline::release() noexcept {
    cudaSetDevice(cfg_.device);
    if (pending_) cudaEventSynchronize(step_end_);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
    if (step_start_) cudaEventDestroy(step_start_);
    if (step_end_) cudaEventDestroy(step_end_);
    for (Slot& s : slots_) {
        cudaFree(s.states);
        cudaFree(s.grad);
        cudaFree(s.param);
    }
    cudaFree(workspace_);
    cudaFree(d_norm_);
    cudaFree(d_nonfinite_);
    cudaFreeHost(h_norm_);
    cudaFreeHost(h_nonfinite_);
    if (h2d_) cudaStreamDestroy(h2d_);
    if (d2h_) cudaStreamDestroy(d2h_);
    if (opt_) cudaStreamDestroy(opt_);
    events_.clear();
    slots_.clear();
    step_start_ = step_end_ = nullptr;
    workspace_ = nullptr;
    d_norm_ = nullptr;
    d_nonfinite_ = nullptr;
    h_norm_ = nullptr;
    h_nonfinite_ = nullptr;
    h2d_ = d2h_ = opt_ = nullptr;
    pending_ = false;
}

void ChunkPipeline::ensure_events(std::uint32_t count) {
    const std::size_t need = static_cast<std::size_t>(count) * kEvPerChunk;
    while (events_.size() < need) {
        cudaEvent_t e;
        check_cuda(cudaEventCreate(&e), "event");
        events_.push_back(e);
    }
}

void ChunkPipeline::issue_h2d(std::uint32_t i) {
    const fy_chunk& c = chunks_[i];
    const std::uint32_t S = static_cast<std::uint32_t>(slots_.size());
    Slot& slot = slots_[i % S];
    if (i >= S) check_cuda(cudaStreamWaitEvent(h2d_, ev(i - S, kD2hEnd), 0), "wait slot");
    if (i >= 2) check_cuda(cudaStreamWaitEvent(h2d_, ev(i - 2, kUpdEnd), 0), "wait read gate");
    check_cuda(cudaEventRecord(ev(i, kH2dStart), h2d_), "record");
    if (!resident(c)) {
        const std::uint64_t stride = c.states_stride ? c.states_stride : c.n;
        if (stride == c.n)
            check_cuda(cudaMemcpyAsync(slot.states, c.h_states, 12ull * c.n, cudaMemcpyHostToDevice,
                                       h2d_),
                       "H2D states");
        else  // master, m, v rows of a strided SoA -> contiguous slot (one copy per
              // row: 2D copies cap the pitch, and a 175B block's rows are 7 GB apart)
            for (int r = 0; r < 3; ++r)
                check_cuda(cudaMemcpyAsync(slot.states + 4 * c.n * r,
                                           static_cast<const float*>(c.h_states) + stride * r, 4 * c.n,
                                           cudaMemcpyHostToDevice, h2d_),
                           "H2D states (strided)");
    }
    if (cfg_.grads_on_host)
        check_cuda(cudaMemcpyAsync(slot.grad, c.grad, std::uint64_t(grad_bytes_) * c.n,
                                   cudaMemcpyHostToDevice, h2d_),
                   "H2D grads");
    check_cuda(cudaEventRecord(ev(i, kH2dEnd), h2d_), "record");
}

void ChunkPipeline::issue_update(std::uint32_t i) {
    const fy_chunk& c = chunks_[i];
    Slot& slot = slots_[i % slots_.size()];
    check_cuda(cudaStreamWaitEvent(opt_, ev(i, kH2dEnd), 0), "wait state read");
    if (c.grad_ready)
        check_cuda(cudaStreamWaitEvent(opt_, static_cast<cudaEvent_t>(c.grad_ready), 0),
                   "wait grad");
    check_cuda(cudaEventRecord(ev(i, kUpdStart), opt_), "record");
    AdamLaunch a{};
    float* states = reinterpret_cast<float*>(resident(c) ? c.h_states : slot.states);
    // staged slots are contiguous; device-resident states keep the caller's stride
    const std::uint64_t stride = resident(c) && c.states_stride ? c.states_stride : c.n;
    a.master = states;
    a.m = states + stride;
    a.v = states + 2 * stride;
    a.grad = cfg_.grads_on_host ? slot.grad : c.grad;
    a.grad_dtype = cfg_.grad_dtype;
    a.param = cfg_.keep_params_on_device ? c.d_param : (cfg_.params_to_host ? slot.param : nullptr);
    a.param_dtype = cfg_.param_dtype;
    a.n = c.n;
    // one DeepSpeed adam_update per chunk: the counter advances per chunk
    fy_adam_hparams hp = unit_hp_ ? unit_hp_[i] : hp_;
    if (!cfg_.no_step_counter && !hp.beta_t_given) {
        counter_.increment(hp.step, hp.beta1, hp.beta2);
        hp.beta_t_given = 1;
        hp.beta1_t = counter_.beta1_t;
        hp.beta2_t = counter_.beta2_t;
    }
    a.s = scalars_of(hp);
    a.s.scale_dev = scale_dev_;  // a skipped update still writes params from master
    a.s.skip_dev = skip_dev_;
    a.grad_sq_sum = want_norm_ ? d_norm_ : nullptr;
    a.accumulate_sq = 1;
    a.workspace = workspace_;
    a.nonfinite = d_nonfinite_;
    check_cuda(launch_adamw(a, opt_), "adamw launch");
    check_cuda(cudaEventRecord(ev(i, kUpdEnd), opt_), "record");
    if (c.update_done)
        check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(c.update_done), opt_), "record update_done");
}

void ChunkPipeline::issue_d2h(std::uint32_t i) {
    const fy_chunk& c = chunks_[i];
    Slot& slot = slots_[i % slots_.size()];
    check_cuda(cudaStreamWaitEvent(d2h_, ev(i, kUpdEnd), 0), "wait update");
    check_cuda(cudaEventRecord(ev(i, kD2hStart), d2h_), "record");
    if (!resident(c)) {
        const std::uint64_t stride = c.states_stride ? c.states_stride : c.n;
        if (stride == c.n)
            check_cuda(cudaMemcpyAsync(c.h_states, slot.states, 12ull * c.n, cudaMemcpyDeviceToHost,
                                       d2h_),
                       "D2H states");
        else
            for (int r = 0; r < 3; ++r)
                check_cuda(cudaMemcpyAsync(static_cast<float*>(c.h_states) + stride * r,
                                           slot.states + 4 * c.n * r, 4 * c.n, cudaMemcpyDeviceToHost, d2h_),
                           "D2H states (strided)");
    }
    if (cfg_.params_to_host) {
        const void* src = cfg_.keep_params_on_device ? c.d_param : slot.param;
        check_cuda(cudaMemcpyAsync(c.h_param, src, std::uint64_t(param_bytes_) * c.n,
                                   cudaMemcpyDeviceToHost, d2h_),
                   "D2H params");
    }
    check_cuda(cudaEventRecord(ev(i, kD2hEnd), d2h_), "record");
}

void ChunkPipeline::step(const fy_chunk* chunks, std::uint32_t count, const fy_adam_hparams& hp,
                         bool want_norm, const fy_adam_hparams* per_chunk_hp, cudaEvent_t start_after) {
    if (pending_) throw ArgError("pipeline: previous step not waited");
    if (count == 0) throw ArgError("pipeline: empty step");
    for (std::uint32_t i = 0; i < count; ++i) {
        const fy_chunk& c = chunks[i];
        if (c.n == 0 || c.n > cfg_.max_chunk_elems)
            throw ArgError("pipeline: chunk " + std::to_string(i) + " size out of range");
        if (!c.h_states || !c.grad) throw ArgError("pipeline: chunk missing states or grad");
        if (c.states_stride != 0 && c.states_stride < c.n)
            throw ArgError("pipeline: chunk " + std::to_string(i) + " states_stride < n");
        if (cfg_.params_to_host && !c.h_param) throw ArgError("pipeline: chunk missing h_param");
        if (cfg_.keep_params_on_device && !c.d_param)
            throw ArgError("pipeline: chunk missing d_param");
    }
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    ensure_events(count);
    chunks_ = chunks;
    want_norm_ = want_norm;
    hp_ = hp;
    unit_hp_ = per_chunk_hp;

    // Step boundary: the previous step's write-backs own the slots.
    if (have_prev_) check_cuda(cudaStreamWaitEvent(h2d_, step_end_, 0), "wait prev");
    if (start_after) check_cuda(cudaStreamWaitEvent(h2d_, start_after, 0), "wait start_after");
    check_cuda(cudaEventRecord(step_start_, h2d_), "record");
    check_cuda(cudaStreamWaitEvent(opt_, step_start_, 0), "wait start");
    check_cuda(cudaMemsetAsync(d_norm_, 0, sizeof(double), opt_), "memset");
    check_cuda(cudaMemsetAsync(d_nonfinite_, 0, sizeof(int), opt_), "memset");

    issue_h2d(0);
    for (std::uint32_t i = 0; i < count; ++i) {
        issue_update(i);
        issue_d2h(i);
        if (i + 1 < count) issue_h2d(i + 1);
    }
    check_cuda(cudaStreamWaitEvent(d2h_, ev(count - 1, kUpdEnd), 0), "wait");
    check_cuda(cudaMemcpyAsync(h_norm_, d_norm_, sizeof(double), cudaMemcpyDeviceToHost, d2h_), "norm");
    check_cuda(cudaMemcpyAsync(h_nonfinite_, d_nonfinite_, sizeof(int), cudaMemcpyDeviceToHost, d2h_),
               "flag");
    check_cuda(cudaEventRecord(step_end_, d2h_), "record");
    chunks_ = nullptr;
    unit_hp_ = nullptr;
    pending_ = true;
    have_prev_ = true;
    last_count_ = count;
}

void ChunkPipeline::wait(double* grad_sq_sum, int* nonfinite) {
    if (!pending_) throw ArgError("pipeline: no step in flight");
    check_cuda(cudaEventSynchronize(step_end_), "step completion");
    pending_ = false;
    if (grad_sq_sum) *grad_sq_sum = want_norm_ ? *h_norm_ : 0.0;
    if (nonfinite) *nonfinite = *h_nonfinite_;
}

void ChunkPipeline::timings(fy_chunk_timing* out, std::uint32_t count, std::uint64_t* step_ns) const {
    if (pending_) throw ArgError("pipeline: step still in flight");
    if (count > last_count_) throw ArgError("pipeline: more timings requested than chunks");
    auto ns = [&](cudaEvent_t e) {
        float ms = 0.0f;
        check_cuda(cudaEventElapsedTime(&ms, step_start_, e), "elapsed");
        return static_cast<std::uint64_t>(static_cast<double>(ms) * 1e6 + 0.5);
    };
    for (std::uint32_t i = 0; i < count; ++i) {
        out[i].h2d_start_ns = ns(ev(i, kH2dStart));
        out[i].h2d_end_ns = ns(ev(i, kH2dEnd));
        out[i].upd_start_ns = ns(ev(i, kUpdStart));
        out[i].upd_end_ns = ns(ev(i, kUpdEnd));
        out[i].d2h_start_ns = ns(ev(i, kD2hStart));
        out[i].d2h_end_ns = ns(ev(i, kD2hEnd));
    }
    if (step_ns) *step_ns = ns(step_end_);
}

} // namespace fy
