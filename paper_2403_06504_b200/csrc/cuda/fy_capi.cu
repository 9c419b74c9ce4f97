// C ABI of the B200 optimizer path (include/fuyou/fy_adam.h).
// Error handling mirrors the reference C ABI (proj/src/capi.cpp:19-51):
// thread-local last error, every body wrapped so no exception escapes.

#include "fuyou/fy_adam.h"

#include "adamw_kernels.cuh"
#include "pipeline.cuh"
#include "shard.cuh"
#include "swap.cuh"

#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_fy_error;

fy_status fail(fy_status code, const std::string& msg) {
    g_fy_error = msg;
    return code;
}

template <typename Fn>
fy_status guard(Fn&& fn) {
    try {
        return fn();
    } catch (const fy::ArgError& e) {
        return fail(FY_ERR_CONFIG, e.what());
    } catch (const fy::DeviceError& e) {
        return fail(FY_ERR_DEVICE, e.what());
    } catch (const std::bad_alloc&) {
        return fail(FY_ERR_INFEASIBLE, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(FY_ERR_INTERNAL, e.what());
    } catch (...) {
        return fail(FY_ERR_INTERNAL, "unknown error");
    }
}

bool valid_grad_dtype(int d) { return d == FY_BF16 || d == FY_FP16 || d == FY_FP32; }
bool valid_param_dtype(int d) { return d == FY_BF16 || d == FY_FP16; }

} // namespace

namespace {
fy_status fy_adamw_chunk_impl(const fy_adamw_args* a, void* stream, const fy::Peers* peers);
} // namespace

struct fy_pipeline {
    explicit fy_pipeline(const fy_pipeline_config& c) : impl(c) {}
    fy::ChunkPipeline impl;
};

extern "C" {

const char* fy_version(void) { return "0.1.0-b200"; }

const char* fy_last_error(void) { return g_fy_error.c_str(); }

uint32_t fy_adamw_workspace_floats(void) { return fy::kWorkspaceFloats; }

fy_status fy_adamw_chunk(const fy_adamw_args* a, void* stream) {
    if (!a) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] { return fy_adamw_chunk_impl(a, stream, nullptr); });
}

fy_status fy_clip_coef(const double* grad_sq_sum, const int* nonfinite, float max_norm,
                       float* scale_out, int* skip_out, void* stream) {
    if (!grad_sq_sum || (!scale_out && !skip_out)) return fail(FY_ERR_CONFIG, "null argument");
    if (!(max_norm >= 0.0f)) return fail(FY_ERR_CONFIG, "max_norm must be >= 0 (0 = no clipping)");
    return guard([&] {
        fy::check_cuda(fy::launch_clip_coef(grad_sq_sum, nonfinite, max_norm, scale_out, skip_out,
                                            static_cast<cudaStream_t>(stream)),
                       "fy_clip_coef");
        return FY_OK;
    });
}

fy_status fy_adamw_chunks(const fy_adamw_args* list, uint32_t count, void* stream) {
    if (!list && count > 0) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        std::vector<fy::AdamLaunch> ls;
        ls.reserve(count);
        for (uint32_t i = 0; i < count; ++i) {
            const fy_adamw_args* a = &list[i];
            const fy_adamw_args* f = &list[0];
            const std::string at = "chunk " + std::to_string(i) + ": ";
            if (a->n > 0 && (!a->master || !a->exp_avg || !a->exp_avg_sq || !a->grad))
                return fail(FY_ERR_CONFIG, at + "null argument");
            if (!valid_grad_dtype(a->grad_dtype)) return fail(FY_ERR_CONFIG, at + "bad grad_dtype");
            if (a->param_out && !valid_param_dtype(a->param_dtype))
                return fail(FY_ERR_CONFIG, at + "param_dtype must be bf16 or fp16");
            if (a->param_out && a->param_out == a->grad && a->grad_dtype == FY_FP32)
                return fail(FY_ERR_CONFIG, at + "param_out may alias grad only for 16-bit grads");
            if (a->grad_sq_sum && !a->workspace) return fail(FY_ERR_CONFIG, at + "grad_sq_sum requires workspace");
            if (a->hp.step == 0) return fail(FY_ERR_CONFIG, at + "step must be >= 1");
            if (a->grad_dtype != f->grad_dtype || (a->param_out != nullptr) != (f->param_out != nullptr) ||
                (a->param_out && a->param_dtype != f->param_dtype))
                return fail(FY_ERR_CONFIG, at + "dtypes / param_out presence differ from chunk 0");
            if (a->grad_sq_sum != f->grad_sq_sum || a->workspace != f->workspace ||
                a->nonfinite_flag != f->nonfinite_flag || a->accumulate_sq != f->accumulate_sq)
                return fail(FY_ERR_CONFIG, at + "statistics outputs differ from chunk 0");
            if (a->n == 0) continue;
            fy::AdamLaunch l{};
            l.master = a->master;
            l.m = a->exp_avg;
            l.v = a->exp_avg_sq;
            l.grad = a->grad;
            l.grad_dtype = a->grad_dtype;
            l.param = a->param_out;
            l.param_dtype = a->param_dtype;
            l.n = a->n;
            l.s = fy::scalars_of(a->hp);
            l.grad_sq_sum = a->grad_sq_sum;
            l.accumulate_sq = a->accumulate_sq;
            l.workspace = a->workspace;
            l.nonfinite = a->nonfinite_flag;
            if (a->grad_scale_dev != f->grad_scale_dev || a->skip_if_set != f->skip_if_set)
                return fail(FY_ERR_CONFIG, at + "device-side controls differ from chunk 0");
            l.s.scale_dev = a->grad_scale_dev;
            l.s.skip_dev = a->skip_if_set;
            ls.push_back(l);
        }
        fy::check_cuda(fy::launch_adamw_multi(ls.data(), static_cast<int>(ls.size()),
                                              static_cast<cudaStream_t>(stream)),
                       "fy_adamw_chunks");
        return FY_OK;
    });
}

} // extern "C"

namespace {

// Validation + launch shared by fy_adamw_chunk and fy_adamw_chunk_gather
// (runs inside their guard(); CUDA failures throw fy::DeviceError).
fy_status fy_adamw_chunk_impl(const fy_adamw_args* a, void* stream, const fy::Peers* peers) {
    if (a->n > 0 && (!a->master || !a->exp_avg || !a->exp_avg_sq || !a->grad))
        return fail(FY_ERR_CONFIG, "null argument");
    if (!valid_grad_dtype(a->grad_dtype)) return fail(FY_ERR_CONFIG, "bad grad_dtype");
    if (a->param_out && !valid_param_dtype(a->param_dtype))
        return fail(FY_ERR_CONFIG, "param_dtype must be bf16 or fp16");
    if (a->param_out && a->param_out == a->grad && a->grad_dtype == FY_FP32)
        return fail(FY_ERR_CONFIG, "param_out may alias grad only for 16-bit grads");
    if (a->grad_sq_sum && !a->workspace)
        return fail(FY_ERR_CONFIG, "grad_sq_sum requires workspace");
    if (a->hp.step == 0) return fail(FY_ERR_CONFIG, "step must be >= 1");
    fy::AdamLaunch l{};
    l.master = a->master;
    l.m = a->exp_avg;
    l.v = a->exp_avg_sq;
    l.grad = a->grad;
    l.grad_dtype = a->grad_dtype;
    l.param = a->param_out;
    l.param_dtype = a->param_dtype;
    l.n = a->n;
    l.s = fy::scalars_of(a->hp);
    l.grad_sq_sum = a->grad_sq_sum;
    l.accumulate_sq = a->accumulate_sq;
    l.workspace = a->workspace;
    l.nonfinite = a->nonfinite_flag;
    l.s.scale_dev = a->grad_scale_dev;
    l.s.skip_dev = a->skip_if_set;
    if (peers) l.peers = *peers;
    fy::check_cuda(fy::launch_adamw(l, static_cast<cudaStream_t>(stream)), "fy_adamw_chunk");
    return FY_OK;
}

} // namespace

extern "C" {

fy_status fy_adamw_chunk_gather(const fy_adamw_args* a, void* const* dst, uint32_t ndst, void* stream) {
    if (!a || (ndst > 0 && !dst)) return fail(FY_ERR_CONFIG, "null argument");
    if (ndst > static_cast<uint32_t>(fy::kMaxPeers)) return fail(FY_ERR_CONFIG, "at most 8 destinations");
    if (!a->param_out) return fail(FY_ERR_CONFIG, "fused gather needs param_out (the local copy)");
    return guard([&] {
        for (uint32_t r = 0; r < ndst; ++r)
            if (!dst[r]) return fail(FY_ERR_CONFIG, "null destination");
        fy::Peers peers{};
        peers.count = static_cast<int>(ndst);
        for (uint32_t r = 0; r < ndst; ++r) peers.ptr[r] = dst[r];
        return fy_adamw_chunk_impl(a, stream, &peers);
    });
}

fy_status fy_grad_stats(const void* grad, int grad_dtype, uint64_t n, float grad_scale,
                        double* grad_sq_sum, int accumulate_sq, float* workspace,
                        int* nonfinite_flag, void* stream) {
    if (n > 0 && !grad) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        if (!valid_grad_dtype(grad_dtype)) return fail(FY_ERR_CONFIG, "bad grad_dtype");
        if (grad_sq_sum && !workspace) return fail(FY_ERR_CONFIG, "grad_sq_sum requires workspace");
        fy::check_cuda(fy::launch_grad_stats(grad, grad_dtype, n, grad_scale, grad_sq_sum,
                                             accumulate_sq, workspace, nonfinite_flag,
                                             static_cast<cudaStream_t>(stream)),
                       "fy_grad_stats");
        return FY_OK;
    });
}

fy_status fy_device_info(int device, int* sm_count, int* ctas_per_sm, int* threads_per_cta) {
    if (!sm_count || !ctas_per_sm || !threads_per_cta) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        int ndev = 0;
        fy::check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) return fail(FY_ERR_CONFIG, "no such device");
        int prev = 0;
        fy::check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
        fy::check_cuda(cudaSetDevice(device), "cudaSetDevice");
        const fy::Geometry g = fy::geometry(device);
        cudaSetDevice(prev);
        *sm_count = g.sm_count;
        *ctas_per_sm = g.ctas_per_sm;
        *threads_per_cta = fy::kThreads;
        return FY_OK;
    });
}

fy_status fy_shard_range(uint64_t n, uint32_t world, uint32_t rank, uint32_t align,
                         uint64_t* offset, uint64_t* count) {
    if (!offset || !count) return fail(FY_ERR_CONFIG, "null argument");
    if (world == 0 || rank >= world) return fail(FY_ERR_CONFIG, "rank out of range");
    if (align == 0) align = 1;
    // Equal slices rounded up to `align`; the tail rank takes the remainder
    // (possibly empty when n is small).
    const uint64_t per = (n + world - 1) / world;
    const uint64_t slice = (per + align - 1) / align * align;
    const uint64_t begin = std::min<uint64_t>(n, slice * rank);
    const uint64_t end = std::min<uint64_t>(n, slice * (rank + 1ull));
    *offset = begin;
    *count = end - begin;
    return FY_OK;
}

fy_status fy_pipeline_create(const fy_pipeline_config* cfg, fy_pipeline** out) {
    if (!cfg || !out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        *out = new fy_pipeline(*cfg);
        return FY_OK;
    });
}

void fy_pipeline_destroy(fy_pipeline* p) { delete p; }

fy_status fy_pipeline_step(fy_pipeline* p, const fy_chunk* chunks, uint32_t count,
                           const fy_adam_hparams* hp, int want_grad_norm) {
    if (!p || !chunks || !hp) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        if (hp->step == 0) return fail(FY_ERR_CONFIG, "step must be >= 1");
        p->impl.step(chunks, count, *hp, want_grad_norm != 0);
        return FY_OK;
    });
}

fy_status fy_pipeline_wait(fy_pipeline* p, double* grad_sq_sum, int* nonfinite) {
    if (!p) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        p->impl.wait(grad_sq_sum, nonfinite);
        return FY_OK;
    });
}

fy_status fy_pipeline_set_controls(fy_pipeline* p, const float* grad_scale_dev, const int* skip_if_set) {
    if (!p) return fail(FY_ERR_CONFIG, "null argument");
    p->impl.set_controls(grad_scale_dev, skip_if_set);
    return FY_OK;
}

fy_status fy_pipeline_timings(const fy_pipeline* p, fy_chunk_timing* out, uint32_t count,
                              uint64_t* step_ns) {
    if (!p || (!out && count > 0)) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        p->impl.timings(out, count, step_ns);
        return FY_OK;
    });
}

struct fy_shard {
    explicit fy_shard(const fy_shard_config& c) : impl(c) {}
    fy::ShardGroup impl;
};

fy_status fy_nccl_unique_id(void* id_out) {
    if (!id_out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        fy::nccl_unique_id(id_out);
        return FY_OK;
    });
}

fy_status fy_shard_create(const fy_shard_config* cfg, fy_shard** out) {
    if (!cfg || !out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        *out = new fy_shard(*cfg);
        return FY_OK;
    });
}

void fy_shard_destroy(fy_shard* s) { delete s; }

fy_status fy_shard_slice_info(const fy_shard* s, uint32_t chunk, fy_shard_slice* out) {
    if (!s || !out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.slice_info(chunk, out);
        return FY_OK;
    });
}

fy_status fy_shard_arena(const fy_shard* s, void** base, uint64_t* bytes) {
    if (!s || !base || !bytes) return fail(FY_ERR_CONFIG, "null argument");
    *base = s->impl.arena();
    *bytes = s->impl.arena_bytes();
    return FY_OK;
}

fy_status fy_shard_ipc_handle(const fy_shard* s, void* handle_out) {
    if (!s || !handle_out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.ipc_handle(handle_out);
        return FY_OK;
    });
}

fy_status fy_shard_connect(fy_shard* s, const void* handles) {
    if (!s || !handles) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.connect_handles(handles);
        return FY_OK;
    });
}

fy_status fy_shard_connect_ptrs(fy_shard* s, void* const* arenas) {
    if (!s || !arenas) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.connect_ptrs(arenas);
        return FY_OK;
    });
}

fy_status fy_shard_step(fy_shard* s, const fy_shard_io* io, const fy_adam_hparams* hp, int want_grad_norm,
                        void* stream) {
    if (!s || !io || !hp) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.step(io, *hp, want_grad_norm != 0, static_cast<cudaStream_t>(stream));
        return FY_OK;
    });
}

fy_status fy_shard_wait(fy_shard* s, double* grad_sq_sum, int* nonfinite) {
    if (!s) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.wait(grad_sq_sum, nonfinite);
        return FY_OK;
    });
}

fy_status fy_shard_get_stats(const fy_shard* s, fy_shard_stats* out) {
    if (!s || !out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.stats(out);
        return FY_OK;
    });
}

fy_status fy_shard_update_ms(const fy_shard* s, double* chunk_ms, uint32_t count) {
    if (!s || (!chunk_ms && count > 0)) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.update_ms(chunk_ms, count);
        return FY_OK;
    });
}

struct fy_swapper {
    fy::Swapper impl;
    explicit fy_swapper(const fy_swap_config& c) : impl(c) {}
};

fy_status fy_swapper_create(const fy_swap_config* cfg, fy_swapper** out) {
    if (!cfg || !out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        *out = new fy_swapper(*cfg);
        return FY_OK;
    });
}

void fy_swapper_destroy(fy_swapper* s) { delete s; }

fy_status fy_swap_out(fy_swapper* s, const void* dev_src, uint64_t bytes, int placement, void* ready_event,
                      void* src_free_event, uint64_t* handle_out) {
    if (!s || !dev_src || !handle_out) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        *handle_out = s->impl.swap_out(dev_src, bytes, placement, static_cast<cudaEvent_t>(ready_event),
                                       static_cast<cudaEvent_t>(src_free_event));
        return FY_OK;
    });
}

fy_status fy_swap_in(fy_swapper* s, uint64_t handle, void* dev_dst, void* ready_event, void* done_event) {
    if (!s || !dev_dst) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.swap_in(handle, dev_dst, static_cast<cudaEvent_t>(ready_event),
                        static_cast<cudaEvent_t>(done_event));
        return FY_OK;
    });
}

fy_status fy_swap_release(fy_swapper* s, uint64_t handle) {
    if (!s) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.release(handle);
        return FY_OK;
    });
}

fy_status fy_swapper_sync(fy_swapper* s) {
    if (!s) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        s->impl.sync();
        return FY_OK;
    });
}

fy_status fy_swapper_stats(const fy_swapper* s, uint64_t* host_bytes, uint64_t* file_bytes,
                           const char** io_engine) {
    if (!s) return fail(FY_ERR_CONFIG, "null argument");
    if (host_bytes) *host_bytes = s->impl.host_bytes();
    if (file_bytes) *file_bytes = s->impl.file_bytes();
    if (io_engine) *io_engine = s->impl.io_engine();
    return FY_OK;
}

fy_status fy_ipc_alloc(uint64_t bytes, void** ptr, void* handle_out) {
    if (!ptr || !handle_out || bytes == 0) return fail(FY_ERR_CONFIG, "null argument or zero bytes");
    return guard([&] {
        void* p = nullptr;
        const cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaErrorMemoryAllocation)
            return fail(FY_ERR_INFEASIBLE, "device allocation of " + std::to_string(bytes) + " bytes failed");
        fy::check_cuda(e, "cudaMalloc (ipc)");
        cudaIpcMemHandle_t h;
        const cudaError_t he = cudaIpcGetMemHandle(&h, p);
        if (he != cudaSuccess) {
            cudaFree(p);
            fy::check_cuda(he, "cudaIpcGetMemHandle");
        }
        std::memcpy(handle_out, &h, sizeof h);
        *ptr = p;
        return FY_OK;
    });
}

fy_status fy_ipc_open(const void* handle, void** ptr) {
    if (!handle || !ptr) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        fy::check_cuda(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        return FY_OK;
    });
}

fy_status fy_ipc_close(void* ptr) {
    if (!ptr) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        fy::check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
        return FY_OK;
    });
}

fy_status fy_ipc_free(void* ptr) {
    return guard([&] {
        if (ptr) fy::check_cuda(cudaFree(ptr), "cudaFree (ipc)");
        return FY_OK;
    });
}

fy_status fy_host_alloc_on(uint64_t bytes, int numa_node, void** out) {
    if (!out) return fail(FY_ERR_CONFIG, "null argument");
    if (numa_node < -2) return fail(FY_ERR_CONFIG, "numa_node must be >= -2");
    return guard([&] {
        int node = numa_node;
        if (node == -1) {
            int dev = 0;
            fy::check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
            node = fy::device_numa_node(dev);
        }
        void* p = fy::host_alloc(bytes, node == -2 ? -1 : node, nullptr);
        if (!p) {
            // registration refused (e.g. locked-memory limits): plain
            // cudaHostAlloc, still page-locked, first-touch placement
            const cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
            if (e == cudaErrorMemoryAllocation)
                return fail(FY_ERR_INFEASIBLE, "pinned host allocation of " + std::to_string(bytes) +
                                                   " bytes failed");
            fy::check_cuda(e, "cudaHostAlloc");
        }
        *out = p;
        return FY_OK;
    });
}

fy_status fy_host_alloc(uint64_t bytes, void** out) { return fy_host_alloc_on(bytes, -1, out); }

fy_status fy_host_free(void* p) {
    return guard([&] {
        if (p && !fy::host_free(p)) fy::check_cuda(cudaFreeHost(p), "cudaFreeHost");
        return FY_OK;
    });
}

fy_status fy_device_numa_node(int device, int* node) {
    if (!node) return fail(FY_ERR_CONFIG, "null argument");
    return guard([&] {
        *node = fy::device_numa_node(device);
        return FY_OK;
    });
}

fy_status fy_host_numa_node(const void* p, int* node) {
    if (!p || !node) return fail(FY_ERR_CONFIG, "null argument");
    *node = fy::host_numa_node(p);
    return FY_OK;
}

} // extern "C"

extern "C" fy_status fy_adamw_sm_budget(int max_ctas) {
    if (max_ctas < 0) return fail(FY_ERR_CONFIG, "max_ctas must be >= 0 (0 = all SMs)");
    fy::set_max_ctas(max_ctas);
    return FY_OK;
}

extern "C" fy_status fy_adamw_tune(int path, int unroll, int ctas_per_sm) {
    if (path != 0 && path != 1) return fail(FY_ERR_CONFIG, "path must be 0 (LSU) or 1 (TMA bulk)");
    if (path == 0 && unroll != 0 && unroll != 1 && unroll != 2 && unroll != 4 && unroll != 8)
        return fail(FY_ERR_CONFIG, "unroll must be 0, 1, 2, 4 or 8");
    if (ctas_per_sm < 0 || ctas_per_sm > 32) return fail(FY_ERR_CONFIG, "ctas_per_sm out of range");
#ifdef FY_SWEEP_VARIANTS
    // sweep build: 2 stages and 4 consumer warps ("narrow") are selectable too
    if (path == 1 && unroll != 0 && unroll != 2 && unroll != 3 && unroll != 4 && unroll != 6)
        return fail(FY_ERR_CONFIG, "stages must be 0 (auto), 2, 3, 4 or 6");
    if (path == 1 && ctas_per_sm != 0 && ctas_per_sm != 4 && ctas_per_sm != 8 && ctas_per_sm != 16)
        return fail(FY_ERR_CONFIG, "path 1: third argument is the consumer warp count (4, 8 or 16)");
#else
    if (path == 1 && unroll != 0 && unroll != 3 && unroll != 4 && unroll != 6)
        return fail(FY_ERR_CONFIG, "stages must be 0 (auto), 3, 4 or 6");
    if (path == 1 && ctas_per_sm != 0 && ctas_per_sm != 8 && ctas_per_sm != 16)
        return fail(FY_ERR_CONFIG, "path 1: third argument is the consumer warp count (0 = auto, 8, 16)");
#endif
    fy::set_tuning(path, unroll, ctas_per_sm);
    return FY_OK;
}

#ifdef FY_SWEEP_VARIANTS
// Sweep build only (build/sweep/liboffsim_sweep.so): TMA kernel variants
// that are not product configurations (see adamw_kernels.cu dispatch_sweep).
extern "C" fy_status fy_adamw_tune_bulk(int tile, int split, int probe) {
    if (tile != 1024 && tile != 2048 && tile != 4096) return fail(FY_ERR_CONFIG, "tile must be 1024, 2048 or 4096");
    if (split != 0 && split != 1) return fail(FY_ERR_CONFIG, "split must be 0 or 1");
    if (probe < 0 || probe > 6) return fail(FY_ERR_CONFIG, "probe must be 0..6");
    fy::set_bulk_variant(tile, split, probe);
    return FY_OK;
}
#endif

extern "C" fy_status fy_adam_counter_init(fy_adam_counter* c, float beta1, float beta2) {
    if (!c) return fail(FY_ERR_CONFIG, "null argument");
    fy::StepCounter k;
    k.construct(beta1, beta2);
    fy::store_counter(k, c);
    return FY_OK;
}

extern "C" fy_status fy_adam_counter_next(fy_adam_counter* c, fy_adam_hparams* hp) {
    if (!c || !hp) return fail(FY_ERR_CONFIG, "null argument");
    if (hp->step == 0) return fail(FY_ERR_CONFIG, "step must be >= 1");
    fy::StepCounter k = fy::load_counter(*c);
    k.increment(hp->step, hp->beta1, hp->beta2);
    fy::store_counter(k, c);
    hp->beta_t_given = 1;
    hp->beta1_t = k.beta1_t;
    hp->beta2_t = k.beta2_t;
    return FY_OK;
}
