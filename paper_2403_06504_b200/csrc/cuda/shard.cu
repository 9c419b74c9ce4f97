// Sharded optimizer step (fy_shard_*): see shard.cuh for the design.
//
// Reference anchor: the optimizer group block `opt state_s2c gK -> opt update
// gK -> opt state_c2s gK / opt param_c2s gK` (proj/src/task_graph.cpp:
// 453-503), single-GPU in the reference; here every block is
// split into `world` slices updated concurrently by the GPUs of one node, and
// the all-gather of the updated bf16 params is the only
// cross-GPU traffic.

#include "shard.cuh"

#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <string>

namespace fy {

namespace {

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw DeviceError(std::string(what) + ": " + ncclGetErrorString(r) +
                          (r == ncclInvalidUsage ? " (NCCL needs one distinct GPU per rank)" : ""));
}

std::uint64_t round_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

constexpr int kEntry = 0, kExit = 1;
constexpr long long kBarrierTimeoutNs = 120ll * 1000 * 1000 * 1000;  // FY_BARRIER_TIMEOUT_S overrides

long long barrier_timeout_ns() {
    const char* e = std::getenv("FY_BARRIER_TIMEOUT_S");
    const double sec = e ? std::atof(e) : 0.0;
    return sec > 0 ? static_cast<long long>(sec * 1e9) : kBarrierTimeoutNs;
}

struct BarrierArgs {
    unsigned char* peer[kMaxWorld];  // arena base of every rank (peer mappings)
    unsigned char* own;
    int world, rank, kind;
    unsigned long long seq;
    const double* my_norm;           // exchange (exit barrier) when non-null
    const int* my_nonfinite;
    double* total;                   // sum over ranks, in rank order
    int* nonfinite_out;
    int* err;
    long long timeout_ns;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One thread: publish this rank's arrival (and its norm / flag) in every
// rank's arena header, then wait until every rank has published `seq`.
// Every store this rank made to peer memory before this kernel (the update
// kernels' epilogue, the copy engines' pushes on this stream) is ordered
// before the flag by the system-scope fence + release store; a peer's
// acquire load of the flag orders its later reads after them.
__global__ void shard_barrier_kernel(BarrierArgs a) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int r = 0; r < a.world; ++r) {
        auto* h = reinterpret_cast<ArenaHeader*>(a.peer[r]);
        if (a.my_norm) {
            *reinterpret_cast<volatile double*>(&h->norms[a.rank]) = *a.my_norm;
            *reinterpret_cast<volatile int*>(&h->nonfinite[a.rank]) = a.my_nonfinite ? *a.my_nonfinite : 0;
        }
    }
    __threadfence_system();
    for (int r = 0; r < a.world; ++r)
        st_release_sys(&reinterpret_cast<ArenaHeader*>(a.peer[r])->flags[a.kind][a.rank], a.seq);
    auto* own = reinterpret_cast<ArenaHeader*>(a.own);
    const long long t0 = global_ns();
    for (int r = 0; r < a.world; ++r) {
        while (ld_acquire_sys(&own->flags[a.kind][r]) < a.seq) {
            if (global_ns() - t0 > a.timeout_ns) {
                *a.err = 1;  // reported by fy_shard_wait; never hang the GPU
                return;
            }
            __nanosleep(200);
        }
    }
    if (a.my_norm) {
        double s = 0.0;
        int bad = 0;
        for (int r = 0; r < a.world; ++r) {
            s += *reinterpret_cast<volatile double*>(&own->norms[r]);
            bad |= *reinterpret_cast<volatile int*>(&own->nonfinite[r]);
        }
        *a.total = s;
        *a.nonfinite_out = bad;
    }
}

} // namespace

ShardGroup::ShardGroup(const fy_shard_config& cfg) : cfg_(cfg) {
    if (cfg_.world == 0 || cfg_.world > kMaxWorld) throw ArgError("shard: world must be 1..9");
    if (cfg_.rank >= cfg_.world) throw ArgError("shard: rank out of range");
    if (cfg_.chunk_count == 0 || !cfg_.chunk_elems) throw ArgError("shard: no chunks");
    if (cfg_.grad_dtype < FY_BF16 || cfg_.grad_dtype > FY_FP32) throw ArgError("shard: bad grad_dtype");
    if (cfg_.param_dtype != FY_BF16 && cfg_.param_dtype != FY_FP16)
        throw ArgError("shard: param_dtype must be bf16 or fp16");
    if (cfg_.tier != FY_TIER_DEVICE && cfg_.tier != FY_TIER_HOST) throw ArgError("shard: bad tier");
    if (cfg_.gather != FY_GATHER_NONE && cfg_.gather != FY_GATHER_NCCL && cfg_.gather != FY_GATHER_PEER)
        throw ArgError("shard: bad gather");
    // world 1: nothing to gather (an explicit NCCL gather still runs, on a
    // one-rank communicator — the same calls as at world > 1)
    if (cfg_.world == 1 && cfg_.gather == FY_GATHER_PEER) cfg_.gather = FY_GATHER_NONE;
    if (cfg_.world > 1 && cfg_.gather == FY_GATHER_NONE)
        throw ArgError("shard: world > 1 needs a gather (NCCL or PEER)");
    if (cfg_.gather == FY_GATHER_NCCL && !cfg_.nccl_id) throw ArgError("shard: FY_GATHER_NCCL needs nccl_id");
    pbytes_ = 2;
    gbytes_ = cfg_.grad_dtype == FY_FP32 ? 4 : 2;
    const std::uint32_t W = cfg_.world;

    std::uint64_t off = kArenaHeaderBytes, max_piece = 0;
    slices_.resize(cfg_.chunk_count);
    for (std::uint32_t c = 0; c < cfg_.chunk_count; ++c) {
        Slice& s = slices_[c];
        s.n = cfg_.chunk_elems[c];
        if (s.n == 0) throw ArgError("shard: chunk " + std::to_string(c) + " is empty");
        // fy_shard_range with align 8: 128-bit vectors never straddle a slice
        s.stride = round_up((s.n + W - 1) / W, 8);
        const std::uint64_t b = std::min<std::uint64_t>(s.n, s.stride * cfg_.rank);
        const std::uint64_t e = std::min<std::uint64_t>(s.n, s.stride * (cfg_.rank + 1ull));
        s.offset = b;
        s.count = e - b;
        s.arena_off = off;
        off = round_up(off + W * s.stride * pbytes_, 256);
        const std::uint64_t piece = cfg_.piece_elems ? std::min<std::uint64_t>(cfg_.piece_elems, s.count) : s.count;
        max_piece = std::max(max_piece, piece);
    }
    arena_bytes_ = off;

    try {
        check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
        const cudaError_t ae = cudaMalloc(&arena_, arena_bytes_);
        if (ae == cudaErrorMemoryAllocation) {
            (void)cudaGetLastError();
            throw std::bad_alloc();
        }
        check_cuda(ae, "shard arena");
        check_cuda(cudaMemset(arena_, 0, kArenaHeaderBytes), "arena header");
        int lo = 0, hi = 0;
        check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
        check_cuda(cudaStreamCreateWithPriority(&opt_, cudaStreamNonBlocking, hi), "opt stream");
        check_cuda(cudaStreamCreateWithFlags(&comm_s_, cudaStreamNonBlocking), "comm stream");
        check_cuda(cudaEventCreate(&start_), "event");
        check_cuda(cudaEventCreate(&done_), "event");
        check_cuda(cudaEventCreateWithFlags(&upd_all_, cudaEventDisableTiming), "event");
        chunk_ev_.resize(cfg_.chunk_count);
        // chunk_ev_ marks each chunk's end (gather / D2H waits) and, timed,
        // doubles as the next chunk's start for update_ms: one event per
        // chunk on the update stream (each record is a few us of device time
        // between the kernels; r02am: 3 per chunk cost 0.25 ms per 13B step)
        for (cudaEvent_t& e : chunk_ev_) check_cuda(cudaEventCreate(&e), "event");
        upd_t0_.resize(cfg_.chunk_count);  // only after a grad_ready wait
        for (cudaEvent_t& e : upd_t0_) check_cuda(cudaEventCreate(&e), "event");
        check_cuda(cudaEventCreate(&upd_start_), "event");
        t0_recorded_.assign(cfg_.chunk_count, 0);
        // every kernel a step may launch is loaded now, before any device
        // barrier can spin (lazy loading would deadlock behind it)
        const void* anchors[] = {reinterpret_cast<const void*>(shard_barrier_kernel)};
        check_cuda(preload_kernels(anchors, 1), "preload kernels");
        check_cuda(cudaMalloc(&workspace_, sizeof(float) * kWorkspaceFloats), "workspace");
        check_cuda(cudaMalloc(&d_norm_, sizeof(double)), "norm");
        check_cuda(cudaMalloc(&d_total_, sizeof(double)), "norm");
        check_cuda(cudaMalloc(&d_nonfinite_, 2 * sizeof(int)), "flags");
        d_err_ = d_nonfinite_ + 1;
        check_cuda(cudaMemset(d_nonfinite_, 0, 2 * sizeof(int)), "flags");
        check_cuda(cudaHostAlloc(&h_total_, sizeof(double), cudaHostAllocDefault), "host norm");
        check_cuda(cudaHostAlloc(&h_flags_, 2 * sizeof(int), cudaHostAllocDefault), "host flags");
        h_flags_[0] = h_flags_[1] = 0;
        peers_.assign(W, nullptr);
        peers_[cfg_.rank] = arena_;
        if (W == 1) connected_ = true;

        if (cfg_.nccl_id && (W > 1 || cfg_.gather == FY_GATHER_NCCL)) {
            ncclUniqueId id;
            std::memcpy(&id, cfg_.nccl_id, sizeof id);
            check_nccl(ncclCommInitRank(&comm_, static_cast<int>(W), id, static_cast<int>(cfg_.rank)),
                       "ncclCommInitRank");
            if (cfg_.gather == FY_GATHER_PEER) {
                // bootstrap the peer table through the communicator: all-gather
                // every rank's arena IPC handle (64 B each)
                unsigned char* d = nullptr;
                check_cuda(cudaMalloc(&d, W * FY_IPC_HANDLE_BYTES), "handles");
                std::vector<unsigned char> h(W * FY_IPC_HANDLE_BYTES);
                ipc_handle(h.data() + cfg_.rank * FY_IPC_HANDLE_BYTES);
                check_cuda(cudaMemcpy(d + cfg_.rank * FY_IPC_HANDLE_BYTES, h.data() + cfg_.rank * FY_IPC_HANDLE_BYTES,
                                      FY_IPC_HANDLE_BYTES, cudaMemcpyHostToDevice),
                           "handle H2D");
                check_nccl(ncclAllGather(d + cfg_.rank * FY_IPC_HANDLE_BYTES, d, FY_IPC_HANDLE_BYTES, ncclUint8,
                                         comm_, comm_s_),
                           "ncclAllGather (handles)");
                check_cuda(cudaStreamSynchronize(comm_s_), "handle exchange");
                check_cuda(cudaMemcpy(h.data(), d, h.size(), cudaMemcpyDeviceToHost), "handles D2H");
                cudaFree(d);
                connect_handles(h.data());
            }
        }
        if (cfg_.tier == FY_TIER_HOST || cfg_.grads_on_host) {
            // streamed states and / or host gradients: the chunk pipeline
            // moves them (device-tier states stay in place, states_on_device)
            fy_pipeline_config pc{};
            pc.device = cfg_.device;
            pc.max_chunk_elems = std::max<std::uint64_t>(max_piece, 8);
            pc.slots = cfg_.slots ? cfg_.slots : 3;
            pc.grad_dtype = cfg_.grad_dtype;
            pc.param_dtype = cfg_.param_dtype;
            pc.grads_on_host = cfg_.grads_on_host ? 1 : 0;
            pc.params_to_host = cfg_.params_to_host;
            pc.keep_params_on_device = 1;  // the arena is the device copy
            pc.states_on_device = cfg_.tier == FY_TIER_DEVICE ? 1 : 0;
            pc.no_step_counter = 1;        // the shard passes each chunk's beta^t
            pipe_ = std::make_unique<ChunkPipeline>(pc);
        }
    } catch (...) {
        release();
        throw;
    }
}

ShardGroup::~ShardGroup() { release(); }

void ShardGroup::release() noexcept {
    cudaSetDevice(cfg_.device);
    if (pending_ && done_) cudaEventSynchronize(done_);
    pipe_.reset();
    if (comm_) ncclCommDestroy(comm_);
    comm_ = nullptr;
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    opened_.clear();
    for (auto* v : {&chunk_ev_, &upd_t0_}) {
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
        v->clear();
    }
    for (cudaEvent_t* e : {&start_, &done_, &upd_all_, &upd_start_})
        if (*e) cudaEventDestroy(*e), *e = nullptr;
    if (opt_) cudaStreamDestroy(opt_);
    if (comm_s_) cudaStreamDestroy(comm_s_);
    opt_ = comm_s_ = nullptr;
    cudaFree(arena_);
    cudaFree(workspace_);
    cudaFree(d_norm_);
    cudaFree(d_total_);
    cudaFree(d_nonfinite_);
    cudaFreeHost(h_total_);
    cudaFreeHost(h_flags_);
    arena_ = nullptr;
    workspace_ = nullptr;
    d_norm_ = d_total_ = nullptr;
    d_nonfinite_ = d_err_ = nullptr;
    h_total_ = nullptr;
    h_flags_ = nullptr;
    pending_ = false;
}

void ShardGroup::slice_info(std::uint32_t chunk, fy_shard_slice* out) const {
    if (chunk >= slices_.size()) throw ArgError("shard: chunk out of range");
    const Slice& s = slices_[chunk];
    out->offset = s.offset;
    out->count = s.count;
    out->stride = s.stride;
    out->params = arena_ + s.arena_off;
}

void ShardGroup::ipc_handle(void* out) const {
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, arena_), "cudaIpcGetMemHandle (arena)");
    static_assert(sizeof h == FY_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(out, &h, sizeof h);
}

void ShardGroup::connect_handles(const void* handles) {
    if (cfg_.world == 1) return;
    if (connected_) throw ArgError("shard: already connected");
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    const auto* hb = static_cast<const unsigned char*>(handles);
    for (std::uint32_t r = 0; r < cfg_.world; ++r) {
        if (r == cfg_.rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb + r * FY_IPC_HANDLE_BYTES, sizeof h);
        void* p = nullptr;
        check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle (peer arena)");
        opened_.push_back(p);
        peers_[r] = static_cast<unsigned char*>(p);
    }
    connected_ = true;
}

void ShardGroup::connect_ptrs(void* const* arenas) {
    if (cfg_.world == 1) return;
    if (connected_) throw ArgError("shard: already connected");
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    for (std::uint32_t r = 0; r < cfg_.world; ++r) {
        if (!arenas[r]) throw ArgError("shard: null peer arena");
        if (r == cfg_.rank) {
            if (arenas[r] != arena_) throw ArgError("shard: arenas[rank] is not this shard's arena");
            continue;
        }
        cudaPointerAttributes at{};
        check_cuda(cudaPointerGetAttributes(&at, arenas[r]), "peer arena attributes");
        if (at.type != cudaMemoryTypeDevice) throw ArgError("shard: peer arena is not device memory");
        if (at.device != cfg_.device) {  // another GPU in this process: NVLink peer access
            const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else check_cuda(e, "cudaDeviceEnablePeerAccess");
        }
        peers_[r] = static_cast<unsigned char*>(arenas[r]);
    }
    connected_ = true;
}

void ShardGroup::need_connected() const {
    if (!connected_) throw ArgError("shard: FY_GATHER_PEER needs fy_shard_connect / fy_shard_connect_ptrs first");
}

std::uint16_t* ShardGroup::chunk_params(std::uint32_t c, int peer) const {
    return reinterpret_cast<std::uint16_t*>(peers_[peer] + slices_[c].arena_off);
}

fy_adam_hparams ShardGroup::chunk_hp(const fy_adam_hparams& hp) {
    fy_adam_hparams h = hp;
    if (!cfg_.no_step_counter && !h.beta_t_given) {  // one DeepSpeed adam_update per chunk
        counter_.increment(h.step, h.beta1, h.beta2);
        h.beta_t_given = 1;
        h.beta1_t = counter_.beta1_t;
        h.beta2_t = counter_.beta2_t;
    }
    return h;
}

void ShardGroup::barrier(int kind, cudaStream_t s, const double* my_norm, const int* my_bad) {
    BarrierArgs a{};
    for (std::uint32_t r = 0; r < cfg_.world; ++r) a.peer[r] = peers_[r];
    a.own = arena_;
    a.world = static_cast<int>(cfg_.world);
    a.rank = static_cast<int>(cfg_.rank);
    a.kind = kind;
    a.seq = seq_;
    if (my_norm) {
        a.my_norm = my_norm;
        a.my_nonfinite = my_bad;
        a.total = d_total_;
        a.nonfinite_out = d_nonfinite_;
    }
    a.err = d_err_;
    a.timeout_ns = barrier_timeout_ns();
    shard_barrier_kernel<<<1, 32, 0, s>>>(a);
    check_cuda(cudaGetLastError(), "barrier launch");
}

void ShardGroup::gather_chunk(std::uint32_t c, cudaStream_t s) {
    const Slice& sl = slices_[c];
    const std::uint64_t bytes = sl.stride * pbytes_;
    unsigned char* base = arena_ + sl.arena_off;
    if (cfg_.gather == FY_GATHER_NCCL) {
        // in place: this rank's slice sits at rank*stride of the chunk region
        check_nccl(ncclAllGather(base + cfg_.rank * bytes, base, bytes, ncclUint8, comm_, s), "ncclAllGather");
        gather_bytes_ += (cfg_.world - 1) * bytes;
    } else if (cfg_.gather == FY_GATHER_PEER && sl.count > 0) {
        const std::uint64_t own = sl.count * pbytes_;
        for (std::uint32_t r = 0; r < cfg_.world; ++r) {
            if (r == cfg_.rank) continue;
            check_cuda(cudaMemcpyAsync(peers_[r] + sl.arena_off + cfg_.rank * bytes, base + cfg_.rank * bytes, own,
                                       cudaMemcpyDeviceToDevice, s),
                       "peer push");
            gather_bytes_ += own;
        }
    }
}

void ShardGroup::step(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm, cudaStream_t stream) {
    if (pending_) throw ArgError("shard: previous step not waited");
    if (hp.step == 0) throw ArgError("shard: step must be >= 1");
    if (cfg_.gather == FY_GATHER_PEER) need_connected();
    for (std::uint32_t c = 0; c < cfg_.chunk_count; ++c) {
        if (slices_[c].count == 0) continue;
        if (!io[c].states || !io[c].grad)
            throw ArgError("shard: chunk " + std::to_string(c) + " missing states or grad");
        if (cfg_.params_to_host && !io[c].h_param)
            throw ArgError("shard: chunk " + std::to_string(c) + " missing h_param");
    }
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    ++seq_;
    want_norm_ = want_norm;
    gather_bytes_ = h2d_bytes_ = d2h_bytes_ = 0;
    check_cuda(cudaEventRecord(start_, stream), "record start");
    check_cuda(cudaStreamWaitEvent(comm_s_, start_, 0), "wait start");
    if (!pipe_) step_resident(io, hp, want_norm);
    else step_streamed(io, hp, want_norm);
    check_cuda(cudaMemcpyAsync(h_total_, d_total_, sizeof(double), cudaMemcpyDeviceToHost, comm_s_), "norm D2H");
    check_cuda(cudaMemcpyAsync(h_flags_, d_nonfinite_, 2 * sizeof(int), cudaMemcpyDeviceToHost, comm_s_),
               "flags D2H");
    check_cuda(cudaEventRecord(done_, comm_s_), "record done");
    check_cuda(cudaStreamWaitEvent(stream, done_, 0), "caller waits");
    pending_ = true;
}

void ShardGroup::step_resident(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm) {
    check_cuda(cudaStreamWaitEvent(opt_, start_, 0), "wait start");
    check_cuda(cudaMemsetAsync(d_norm_, 0, sizeof(double), opt_), "memset");
    check_cuda(cudaMemsetAsync(d_nonfinite_, 0, sizeof(int), opt_), "memset");
    const bool peer = cfg_.gather == FY_GATHER_PEER;
    if (peer) barrier(kEntry, opt_, nullptr, nullptr);  // every peer may now receive this step's params
    check_cuda(cudaEventRecord(upd_start_, opt_), "record");
    for (std::uint32_t c = 0; c < cfg_.chunk_count; ++c) {
        const Slice& sl = slices_[c];
        const fy_adam_hparams h = chunk_hp(hp);
        t0_recorded_[c] = 0;
        if (io[c].grad_ready) {
            check_cuda(cudaStreamWaitEvent(opt_, static_cast<cudaEvent_t>(io[c].grad_ready), 0), "wait grad");
            // the chunk's time starts when its gradients are ready, not at
            // the previous chunk's end
            check_cuda(cudaEventRecord(upd_t0_[c], opt_), "record");
            t0_recorded_[c] = 1;
        }
        if (sl.count > 0) {
            AdamLaunch a{};
            float* st = static_cast<float*>(io[c].states);
            a.master = st;
            a.m = st + sl.count;
            a.v = st + 2 * sl.count;
            a.grad = io[c].grad;
            a.grad_dtype = cfg_.grad_dtype;
            a.param = chunk_params(c, static_cast<int>(cfg_.rank)) + cfg_.rank * sl.stride;
            a.param_dtype = cfg_.param_dtype;
            a.n = sl.count;
            a.s = scalars_of(h);
            a.grad_sq_sum = want_norm ? d_norm_ : nullptr;
            a.accumulate_sq = 1;
            a.workspace = workspace_;
            a.nonfinite = d_nonfinite_;
            if (peer) {  // fused gather: the epilogue stores into every peer's arena
                for (std::uint32_t r = 0; r < cfg_.world; ++r) {
                    if (r == cfg_.rank) continue;
                    a.peers.ptr[a.peers.count++] = chunk_params(c, static_cast<int>(r)) + cfg_.rank * sl.stride;
                }
                gather_bytes_ += (cfg_.world - 1) * sl.count * pbytes_;
            }
            check_cuda(launch_adamw(a, opt_), "adamw launch (shard)");
        }
        check_cuda(cudaEventRecord(chunk_ev_[c], opt_), "record chunk");
        if (cfg_.gather == FY_GATHER_NCCL) {
            check_cuda(cudaStreamWaitEvent(comm_s_, chunk_ev_[c], 0), "wait chunk");
            gather_chunk(c, comm_s_);
        }
        if (cfg_.params_to_host && sl.count > 0) {
            check_cuda(cudaStreamWaitEvent(comm_s_, chunk_ev_[c], 0), "wait chunk");
            check_cuda(cudaMemcpyAsync(io[c].h_param, chunk_params(c, static_cast<int>(cfg_.rank)) + cfg_.rank * sl.stride,
                                       sl.count * pbytes_, cudaMemcpyDeviceToHost, comm_s_),
                       "params D2H");
            d2h_bytes_ += sl.count * pbytes_;
        }
    }
    if (peer)  // peers' stores into this arena are complete (and the norms exchanged)
        barrier(kExit, opt_, want_norm ? d_norm_ : nullptr, d_nonfinite_);
    check_cuda(cudaEventRecord(upd_all_, opt_), "record");
    check_cuda(cudaStreamWaitEvent(comm_s_, upd_all_, 0), "wait updates");
    if (cfg_.gather == FY_GATHER_NCCL) {
        if (want_norm) {
            check_nccl(ncclAllReduce(d_norm_, d_total_, 1, ncclFloat64, ncclSum, comm_, comm_s_), "ncclAllReduce");
            check_nccl(ncclAllReduce(d_nonfinite_, d_nonfinite_, 1, ncclInt32, ncclMax, comm_, comm_s_),
                       "ncclAllReduce");
        }
    } else if (!peer || !want_norm) {
        check_cuda(cudaMemcpyAsync(d_total_, d_norm_, sizeof(double), cudaMemcpyDeviceToDevice, comm_s_), "norm");
    }
}

void ShardGroup::step_streamed(const fy_shard_io* io, const fy_adam_hparams& hp, bool want_norm) {
    const bool peer = cfg_.gather == FY_GATHER_PEER;
    if (peer) barrier(kEntry, comm_s_, nullptr, nullptr);
    units_.clear();
    unit_hp_.clear();
    unit_chunk_.clear();
    std::vector<bool> has_unit(cfg_.chunk_count, false);
    for (std::uint32_t c = 0; c < cfg_.chunk_count; ++c) {
        const Slice& sl = slices_[c];
        const fy_adam_hparams h = chunk_hp(hp);
        if (sl.count == 0) continue;
        const std::uint64_t piece = cfg_.piece_elems ? std::min<std::uint64_t>(cfg_.piece_elems, sl.count) : sl.count;
        std::uint16_t* own = chunk_params(c, static_cast<int>(cfg_.rank)) + cfg_.rank * sl.stride;
        for (std::uint64_t o = 0; o < sl.count; o += piece) {
            fy_chunk u{};
            u.n = std::min(piece, sl.count - o);
            u.h_states = static_cast<float*>(io[c].states) + o;
            u.states_stride = sl.count;  // a piece of the slice's SoA [master|m|v]
            u.grad = static_cast<const char*>(io[c].grad) + o * gbytes_;
            u.d_param = own + o;
            u.h_param = io[c].h_param ? static_cast<char*>(io[c].h_param) + o * pbytes_ : nullptr;
            u.grad_ready = o == 0 ? io[c].grad_ready : nullptr;
            u.update_done = o + piece >= sl.count ? chunk_ev_[c] : nullptr;
            units_.push_back(u);
            unit_hp_.push_back(h);
            unit_chunk_.push_back(c);
        }
        has_unit[c] = true;
        const std::uint64_t state_b = cfg_.tier == FY_TIER_HOST ? 12 * sl.count : 0;
        h2d_bytes_ += state_b + (cfg_.grads_on_host ? sl.count * gbytes_ : 0);
        d2h_bytes_ += state_b + (cfg_.params_to_host ? sl.count * pbytes_ : 0);
    }
    if (!units_.empty()) {
        pipe_->step(units_.data(), static_cast<std::uint32_t>(units_.size()), hp, want_norm, unit_hp_.data(),
                    start_);
    }
    for (std::uint32_t c = 0; c < cfg_.chunk_count; ++c) {
        if (cfg_.gather == FY_GATHER_NONE) break;
        if (has_unit[c]) check_cuda(cudaStreamWaitEvent(comm_s_, chunk_ev_[c], 0), "wait chunk");
        gather_chunk(c, comm_s_);  // overlaps the next chunks' streaming
    }
    double* norm = units_.empty() ? d_norm_ : pipe_->device_norm();
    int* bad = units_.empty() ? d_nonfinite_ : pipe_->device_nonfinite();
    if (units_.empty()) {
        check_cuda(cudaMemsetAsync(d_norm_, 0, sizeof(double), comm_s_), "memset");
        check_cuda(cudaMemsetAsync(d_nonfinite_, 0, sizeof(int), comm_s_), "memset");
    } else {
        check_cuda(cudaStreamWaitEvent(comm_s_, pipe_->step_end_event(), 0), "wait pipeline");
    }
    if (peer) {
        barrier(kExit, comm_s_, want_norm ? norm : nullptr, bad);
        if (!want_norm) check_cuda(cudaMemcpyAsync(d_total_, norm, sizeof(double), cudaMemcpyDeviceToDevice, comm_s_), "norm");
    } else if (cfg_.gather == FY_GATHER_NCCL && want_norm) {
        check_nccl(ncclAllReduce(norm, d_total_, 1, ncclFloat64, ncclSum, comm_, comm_s_), "ncclAllReduce");
        check_nccl(ncclAllReduce(bad, d_nonfinite_, 1, ncclInt32, ncclMax, comm_, comm_s_), "ncclAllReduce");
    } else {
        check_cuda(cudaMemcpyAsync(d_total_, norm, sizeof(double), cudaMemcpyDeviceToDevice, comm_s_), "norm");
        if (bad != d_nonfinite_)
            check_cuda(cudaMemcpyAsync(d_nonfinite_, bad, sizeof(int), cudaMemcpyDeviceToDevice, comm_s_), "flag");
    }
}

void ShardGroup::wait(double* grad_sq_sum, int* nonfinite) {
    if (!pending_) throw ArgError("shard: no step in flight");
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    check_cuda(cudaEventSynchronize(done_), "shard step completion");
    pending_ = false;
    if (pipe_) pipe_->mark_waited();
    float ms = 0.0f;
    check_cuda(cudaEventElapsedTime(&ms, start_, done_), "elapsed");
    last_step_ms_ = ms;
    if (h_flags_[1]) throw DeviceError("shard: peer barrier timed out (a rank did not reach the step)");
    if (grad_sq_sum) *grad_sq_sum = want_norm_ ? *h_total_ : 0.0;
    if (nonfinite) *nonfinite = h_flags_[0];
}

void ShardGroup::update_ms(double* out, std::uint32_t count) const {
    if (pending_) throw ArgError("shard: step still in flight");
    if (count > cfg_.chunk_count) throw ArgError("shard: more chunks requested than the shard has");
    for (std::uint32_t c = 0; c < count; ++c) out[c] = 0.0;
    if (seq_ == 0) return;
    if (!pipe_) {
        // chunk c ran from the previous chunk's end (or the step's start,
        // or its grad_ready) to its own end: its update + norm reduction
        cudaEvent_t prev = upd_start_;
        for (std::uint32_t c = 0; c < count; ++c) {
            if (t0_recorded_[c]) prev = upd_t0_[c];
            float ms = 0.0f;
            check_cuda(cudaEventElapsedTime(&ms, prev, chunk_ev_[c]), "elapsed");
            if (slices_[c].count > 0) out[c] = ms;
            prev = chunk_ev_[c];
        }
    } else if (!units_.empty()) {
        std::vector<fy_chunk_timing> t(units_.size());
        std::uint64_t total = 0;
        pipe_->timings(t.data(), static_cast<std::uint32_t>(t.size()), &total);
        for (std::size_t u = 0; u < t.size(); ++u)
            if (unit_chunk_[u] < count) out[unit_chunk_[u]] += (t[u].upd_end_ns - t[u].upd_start_ns) * 1e-6;
    }
}

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    check_nccl(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof id == FY_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof id);
}

void ShardGroup::stats(fy_shard_stats* out) const {
    out->step_ms = last_step_ms_;
    out->gather_bytes = gather_bytes_;
    out->h2d_bytes = h2d_bytes_;
    out->d2h_bytes = d2h_bytes_;
    out->world = cfg_.world;
    out->rank = cfg_.rank;
    out->gather = cfg_.gather;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg_.device);
    const int n_sms = sms > 0 ? sms : 148;
    out->stages = cfg_.grad_dtype != FY_FP32 && budgeted_split(n_sms) ? 6 : tma_stages(n_sms);
    out->consumer_warps = tma_consumer_warps(sms > 0 ? sms : 148, cfg_.grad_dtype == FY_FP32);
}

} // namespace fy
