// B200 graph executor: runs every task of the tier-mapped graph on real
// engines and returns the real SimTrace (include/offsim/exec.hpp).
//
// Lanes -> engines (one CUDA stream each, so every lane is serial, as the
// reference's lane model and check_trace_invariants require):
//   gpu_compute  synthetic fwd/bwd compute (timed kernel, work / rate)
//   cpu_compute  the optimizer lane: fused AdamW kernel (fy::launch_adamw)
//   link_c2g     H2D copy engine      link_g2c   D2H copy engine
//   link_ssd     file tier: pread/pwrite (O_DIRECT) in stream host callbacks
//                host tier: no bytes (zero-length tasks)
// Each task is bracketed by two CUDA events on its lane stream; a task waits
// on the end events of its dependencies on other lanes. Tasks are issued in
// the start order of simulate(mapped graph, measured B200 rates), so each
// engine executes the planned order and every awaited event has already been
// recorded when the wait is enqueued.

#include "adamw_kernels.cuh"
#include "pipeline.cuh"
#include "../core/io_engine.hpp"

#include "offsim/errors.hpp"
#include "offsim/exec.hpp"

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <set>
#include <thread>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>

namespace offsim {

namespace {

using fy::check_cuda;

constexpr std::uint64_t kAlign = 4096;
std::uint64_t round_up(std::uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// ------------------------------------------------------------ kernels

__global__ void spin_kernel(std::uint64_t ns) {
    std::uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Deterministic byte pattern for activation / checkpoint buffers.
__global__ void fill_pattern(std::uint64_t* p, std::uint64_t words, std::uint64_t seed) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < words;
         i += std::uint64_t(gridDim.x) * blockDim.x)
        p[i] = mix64(seed ^ (i * 0x100000001b3ull));
}

// Synthetic optimizer state: master ~ U(-0.02,0.02)-ish, m small, v >= 0,
// bf16 grads ~ 1e-3 (shape of SURVEY.md §8d; exact distribution irrelevant).
__global__ void fill_states(float* st, std::uint64_t n, std::uint64_t seed) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint64_t r = mix64(seed ^ i);
        const float u0 = float(r & 0xffffff) / 16777216.0f - 0.5f;
        const float u1 = float((r >> 24) & 0xffffff) / 16777216.0f - 0.5f;
        st[i] = 0.04f * u0;
        st[n + i] = 2e-3f * u1;
        st[2 * n + i] = 1e-6f * (u0 * u0 + 1e-3f);
    }
}

__global__ void fill_grads(std::uint16_t* g, std::uint64_t n, std::uint64_t seed) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const float u = float(mix64(seed ^ (i + 0x51ed27)) & 0xffffff) / 16777216.0f - 0.5f;
        const float f = 2e-3f * u;
        g[i] = static_cast<std::uint16_t>(__float_as_uint(f) >> 16);
    }
}

__global__ void count_mismatch(const std::uint64_t* a, const std::uint64_t* b, std::uint64_t words,
                               unsigned long long* bad) {
    unsigned long long local = 0;
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < words;
         i += std::uint64_t(gridDim.x) * blockDim.x)
        local += a[i] != b[i];
    if (local) atomicAdd(bad, local);
}

// --------------------------------------------------------- file tier

struct IoRequest {
    fy::IoEngine* io = nullptr;
    fy::IoEngine::Stripe file{}; // the tier file's device files
    void* buf = nullptr;
    std::uint64_t bytes = 0; // rounded to kAlign for O_DIRECT
    std::uint64_t offset = 0;
    bool write = false;
    bool poison_after = false; // overwrite the host buffer after a write
    std::atomic<int>* error = nullptr;
    std::string* error_text = nullptr;
    std::mutex* error_mu = nullptr;
};

// Released at the end of every IO host function, acquired after the device
// synchronisations that wait for them (the CUDA-guaranteed ordering made
// explicit for the C++ memory model and ThreadSanitizer).
std::atomic<std::uint64_t> g_io_done{0};

void CUDART_CB run_io(void* arg) {
    struct Done {
        ~Done() { g_io_done.fetch_add(1, std::memory_order_release); }
    } done;
    auto* r = static_cast<IoRequest*>(arg);
    std::string err;
    try {  // nothing may escape a CUDA host callback
        err = r->io->transfer(r->file, r->buf, r->bytes, r->offset, r->write);
    } catch (const std::exception& e) {
        err = std::string("file tier IO: ") + e.what();
    } catch (...) {
        err = "file tier IO: unknown exception";
    }
    if (!err.empty()) {
        std::lock_guard<std::mutex> lk(*r->error_mu);
        r->error->store(1);
        *r->error_text = err;
        return;
    }
    if (r->write && r->poison_after) {
        // verification: the host copy must not survive to the restore, or a
        // read that never happened would look correct. Every request piece
        // is >= 4 KiB and 4 KiB aligned, so overwriting the first 64 B of
        // every 4 KiB page makes any piece that is not read back differ;
        // a full memset cost ~8 ms per 84 MB checkpoint inside the timed
        // SSD leg (r02o swap sweep).
        auto* p = static_cast<unsigned char*>(r->buf);
        for (std::uint64_t off = 0; off < r->bytes; off += 4096)
            std::memset(p + off, 0xA5, std::min<std::uint64_t>(64, r->bytes - off));
    }
}

// One logical tier file, striped RAID-0 over one file per directory (one
// directory per SSD: the reference's n_ssd devices, hardware.cpp:39-42) in
// kStripeUnit pieces; a single directory is a plain file.
constexpr std::uint64_t kStripeUnit = 4ull << 20;

class TierFile {
public:
    TierFile(const std::vector<std::string>& dirs, const std::string& name, std::uint64_t size, bool direct) {
        const std::uint64_t count = dirs.size();
        const std::uint64_t units = (size + kStripeUnit - 1) / kStripeUnit;
        const std::uint64_t per_dev = count == 1 ? size : (units + count - 1) / count * kStripeUnit;
        for (const std::string& dir : dirs) {
            const std::string path = dir + "/" + name;
            int flags = O_RDWR | O_CREAT | O_TRUNC;
            if (direct) flags |= O_DIRECT;
            int fd = ::open(path.c_str(), flags, 0600);
            if (fd < 0 && direct) fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
            if (fd < 0) {
                const std::string why = std::strerror(errno);
                close_all();
                throw InfeasibleError("cannot open tier file " + path + ": " + why);
            }
            fds_.push_back(fd);
            paths_.push_back(path);
            if (::ftruncate(fd, static_cast<off_t>(per_dev)) != 0) {
                const std::string why = std::strerror(errno);
                close_all();
                throw InfeasibleError("cannot size tier file " + path + ": " + why);
            }
        }
    }
    ~TierFile() { close_all(); }
    TierFile(const TierFile&) = delete;
    TierFile& operator=(const TierFile&) = delete;
    fy::IoEngine::Stripe stripe() const {
        return {fds_.data(), static_cast<unsigned>(fds_.size()), kStripeUnit};
    }

private:
    void close_all() noexcept {
        for (std::size_t i = 0; i < fds_.size(); ++i) {
            ::close(fds_[i]);
            ::unlink(paths_[i].c_str());
        }
        fds_.clear();
        paths_.clear();
    }
    std::vector<int> fds_;
    std::vector<std::string> paths_;
};

// ------------------------------------------------------------- parsing

struct Parsed {
    std::string phase, what; // "fwd","p_c2g"
    std::uint32_t block = 0;
    int layer = -1; // 0..3 within the block when present
};

Parsed parse_name(const std::string& name) {
    // "<phase> <what> <b|g><k>[ <layer kind>]"
    Parsed p;
    std::istringstream is(name);
    std::string tag, kind;
    is >> p.phase >> p.what >> tag >> kind;
    p.block = static_cast<std::uint32_t>(std::stoul(tag.substr(1)));
    static const char* kKinds[] = {"linear_qkv", "linear_htoh", "linear_hto4h", "linear_4htoh"};
    for (int j = 0; j < 4; ++j)
        if (kind == kKinds[j]) p.layer = j;
    return p;
}

struct Pinned {
    void* p = nullptr;
    Pinned() = default;
    explicit Pinned(std::uint64_t bytes) {
        // NUMA-local to the executing GPU (host_mem.cu); cudaHostAlloc if
        // registration is refused
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        bytes = std::max<std::uint64_t>(bytes, kAlign);
        p = fy::host_alloc(bytes, fy::device_numa_node(dev), nullptr);
        if (!p) check_cuda(cudaHostAlloc(&p, bytes, cudaHostAllocPortable), "cudaHostAlloc (executor host buffers)");
    }
    Pinned(Pinned&& o) noexcept : p(o.p) { o.p = nullptr; }
    Pinned& operator=(Pinned&& o) noexcept {
        std::swap(p, o.p);
        return *this;
    }
    ~Pinned() {
        if (p && !fy::host_free(p)) cudaFreeHost(p);
    }
};

struct Device {
    void* p = nullptr;
    Device() = default;
    explicit Device(std::uint64_t bytes) {
        const cudaError_t e = cudaMalloc(&p, std::max<std::uint64_t>(bytes, 256));
        if (e == cudaErrorMemoryAllocation)
            throw InfeasibleError("device allocation of " + std::to_string(bytes) + " bytes failed");
        check_cuda(e, "cudaMalloc (executor)");
    }
    Device(Device&& o) noexcept : p(o.p) { o.p = nullptr; }
    Device& operator=(Device&& o) noexcept {
        std::swap(p, o.p);
        return *this;
    }
    ~Device() {
        if (p) cudaFree(p);
    }
};

// --------------------------------------------------------------- engine

class Engine {
public:
    Engine(const ModelConfig& model, const SwapPlan& plan, const TaskGraph& mapped,
           const ExecOptions& opt, const std::vector<ChunkBuffers>* chunks)
        : model_(model), plan_(plan), g_(mapped), opt_(opt), user_(chunks),
          // one ring for every tier device, io_depth requests in flight on each
          io_(opt.io_depth * static_cast<unsigned>(std::max<std::size_t>(1, opt.file_dirs.size()))) {}

    ~Engine() {
        // drain everything first: host IO callbacks reference io_reqs_ and
        // the staging buffers (matters when a run throws part-way)
        cudaSetDevice(opt_.device);
        for (cudaStream_t s : streams_)
            if (s) cudaStreamSynchronize(s);
        (void)g_io_done.load(std::memory_order_acquire);
        if (blas_) cublasDestroy(blas_);
        for (cudaEvent_t e : events_) cudaEventDestroy(e);
        for (cudaEvent_t e : deps_) cudaEventDestroy(e);
        if (base_) cudaEventDestroy(base_);
        for (cudaStream_t s : streams_)
            if (s) cudaStreamDestroy(s);
    }

    void setup();
    MeasuredRates calibrate();
    const char* io_engine() const { return io_.engine(); }
    std::uint64_t io_registered() const { return io_registered_; }
    std::vector<std::string> file_dirs() const {
        return opt_.file_dirs.empty() ? std::vector<std::string>{opt_.file_dir} : opt_.file_dirs;
    }
    std::uint64_t io_fixed() const { return io_.fixed_requests(); }
    std::uint64_t io_plain() const { return io_.plain_requests(); }
    void run(const SimTrace& planned, ExecReport& rep);
    double warm_file_lane();

private:
    cudaStream_t lane_stream(ResourceId r) const { return streams_[static_cast<int>(r)]; }
    void issue(const Task& t, ExecReport& rep);
    // the file-lane request of a task: tier file, host buffer, bytes, offset
    struct FileOp {
        const TierFile* file = nullptr;
        void* buf = nullptr;
        std::uint64_t bytes = 0, offset = 0;
        bool write = false, poison = false;
    };
    bool file_op(const Task& t, FileOp& op);  // false: not a file request
    void issue_compute(const Task& t, const Parsed& p, cudaStream_t s, bool replay);
    std::uint64_t layer_offset(int j) const; // byte offset of layer j inside the block params

    const ModelConfig& model_;
    const SwapPlan& plan_;
    const TaskGraph& g_;
    ExecOptions opt_;
    const std::vector<ChunkBuffers>* user_;

    std::uint32_t blocks_ = 0;
    std::uint64_t n_ = 0;          // params per block (chunk)
    std::vector<LayerProfile> layers_;
    std::vector<bool> swapped_;
    std::uint64_t ckpt_bytes_ = 0;
    bool file_tier_ = false;
    bool has_update_ = false;
    bool has_weights_ = false;
    // bounded pinned staging rings (file tier, host_ring > 0 or auto)
    bool ring_ = false;
    RingDepths depths_;
    bool acts_on_ssd_ = false;
    std::vector<Pinned> state_ring_, param_ring_, weight_ring_, act_ring_;
    // staging buffers registered with io_uring (READ/WRITE_FIXED requests)
    std::vector<std::pair<void*, std::uint64_t>> io_bufs_;
    std::uint64_t io_registered_ = 0;
    std::map<std::uint32_t, int> ring_slot_; // task id -> ring slot
    std::uint64_t pinned_bytes_ = 0;
    Pinned pin(std::uint64_t bytes) {
        pinned_bytes_ += std::max<std::uint64_t>(bytes, kAlign);
        return Pinned(bytes);
    }
    void* ring_ptr(std::vector<Pinned>& r, std::uint32_t task) { return r[ring_slot_.at(task)].p; }
    void* host_states(std::uint32_t task, std::uint32_t k) {
        return ring_ ? ring_ptr(state_ring_, task) : h_states_[k];
    }
    void* host_params(std::uint32_t task, std::uint32_t k) {
        return ring_ ? ring_ptr(param_ring_, task) : h_params_[k];
    }
    void* host_weights(std::uint32_t task, std::uint32_t k, std::uint64_t layer_off) {
        return ring_ ? ring_ptr(weight_ring_, task) : static_cast<char*>(h_params_[k]) + layer_off;
    }
    void* host_act(std::uint32_t task, const Pinned& unit) {
        return ring_ && acts_on_ssd_ ? ring_ptr(act_ring_, task) : unit.p;
    }
    std::uint64_t checksum_states();
    void assign_ring_slots();

    cudaStream_t streams_[5] = {};
    std::vector<cudaEvent_t> events_;  // [2 id]: start, [2 id + 1]: end (timing)
    std::vector<cudaEvent_t> deps_;    // graph mode: task end, dependency only
    cudaEvent_t base_ = nullptr;
    bool capturing_ = false;           // issue() is being captured into a CUDA graph
    void record_time(cudaEvent_t e, cudaStream_t s) {
        // in a capture an external record becomes an event-record NODE that
        // timestamps when the graph executes (a plain record only marks a
        // capture dependency)
        check_cuda(capturing_ ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s),
                   "record");
    }
    // what a dependent task waits on: zero-work tasks issue no GPU work and
    // no timing event, only their dependency point (deps_); in a capture a
    // plain record is an edge, not a node
    cudaEvent_t end_dep(std::uint32_t id) const {
        return capturing_ || g_.tasks[id].work <= 0.0 ? deps_[id] : events_[2 * id + 1];
    }
    std::vector<std::uint32_t> issued_;  // issue order (each lane's FIFO order)
    bool run_graph(const std::vector<std::pair<std::uint64_t, std::uint32_t>>& order, ExecReport& rep);

    // host side
    std::vector<Pinned> own_states_, own_params_, act_host_, ckpt_host_, grad_host_;
    std::vector<void*> h_states_, h_params_;
    // device side
    std::vector<Device> own_grads_, act_dev_, act_restore_, ckpt_dev_, ckpt_restore_, slots_;
    std::vector<Device> res_states_;  // resident optimizer groups g0..g(R-1): states in HBM
    std::uint32_t resident_ = 0;
    bool is_resident(std::uint32_t k) const { return k < resident_; }

public:
    std::uint32_t resident_count() const { return resident_; }

private:
    void* read_tier_states(std::uint32_t k, Pinned& tmp);  // initial states of chunk k
    void write_back_resident();                             // after the run
    std::vector<const void*> d_grads_;
    Device wscratch_[2];
    int wscratch_turn_ = 0;
    Device workspace_, d_norm_, d_bad_, d_mismatch_;
    int slot_of(std::uint32_t block) const {
        // optimizer groups run in reverse block order: m = blocks - 1 - k
        return static_cast<int>((blocks_ - 1 - block) % slots_.size());
    }

    // file tier
    std::unique_ptr<TierFile> f_states_, f_params_, f_acts_, f_grads_;
    std::uint64_t tier_states_bytes_ = 0;
    std::vector<std::uint64_t> act_file_off_;
    std::vector<std::uint64_t> ckpt_file_off_;
    std::vector<std::unique_ptr<IoRequest>> io_reqs_;
    fy::IoEngine io_;
    std::atomic<int> io_error_{0};
    std::string io_error_text_;
    std::mutex io_mu_;

    fy::AdamScalars scalars_{};
    double compute_rate_ = 0.0;
    // gemm compute mode
    bool gemm_ = false;
    bool dataflow_ = false;  // compute_mode "gemm_dataflow": wgrad GEMMs produce the optimizer's grads
    cublasHandle_t blas_ = nullptr;
    Device gemm_a_, gemm_b_, gemm_c_, gemm_ws_;
    void gemm(cudaStream_t s, int m, int n, int k);
    // dW[in x out] = X^T dY with X = the first tokens x in of gemm_a_, dY =
    // the first tokens x out of gemm_b_ (row-major bf16), written to dst
    void wgrad(cudaStream_t s, int tokens, int in, int out, void* dst);
    double expected_grad_sq_ = 0.0;  // gemm_dataflow self-check
    void layer_dims(int j, int& in, int& out) const {
        const int h = static_cast<int>(model_.hidden_dim);
        static const int kIn[4] = {1, 1, 1, 4}, kOut[4] = {3, 1, 4, 1};
        in = kIn[j] * h;
        out = kOut[j] * h;
    }
};

std::uint64_t Engine::layer_offset(int j) const {
    std::uint64_t off = 0;
    for (int k = 0; k < j; ++k) off += layers_[k].param_bytes;
    return off;
}

void Engine::setup() {
    check_cuda(cudaSetDevice(opt_.device), "cudaSetDevice");
    blocks_ = model_.num_layers;
    n_ = 12ull * model_.hidden_dim * model_.hidden_dim;
    layers_ = build_layer_profiles(model_);
    swapped_.assign(layers_.size(), false);
    for (std::uint32_t i : plan_.swapped_layers) swapped_[i] = true;
    ckpt_bytes_ = footprint(model_).checkpoint_bytes_per_block;
    file_tier_ = opt_.tier == StateTier::file;
    if (model_.param_elem_bytes != 2)
        throw ConfigError("executor: param_elem_bytes must be 2 (bf16 params)");
    if (std::llround(model_.optimizer_state_multiplier) != 6)
        throw ConfigError("executor: optimizer_state_multiplier must be 6 (fp32 master, m, v)");
    if (user_ && user_->size() != blocks_)
        throw ConfigError("executor: expected one ChunkBuffers per block");

    int lo = 0, hi = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priorities");
    for (int r = 0; r < 5; ++r) {
        const int prio = r == static_cast<int>(ResourceId::cpu_compute) ? hi : lo;
        check_cuda(cudaStreamCreateWithPriority(&streams_[r], cudaStreamNonBlocking, prio), "stream");
    }
    events_.resize(2 * g_.tasks.size());
    for (cudaEvent_t& e : events_) check_cuda(cudaEventCreate(&e), "event");
    deps_.resize(g_.tasks.size());
    for (cudaEvent_t& e : deps_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreate(&base_), "event");

    const std::uint64_t state_b = 12 * n_, param_b = 2 * n_;
    const std::uint64_t seed = opt_.seed * 0x9e3779b97f4a7c15ull + 17;
    // Allocate only what the executed graph touches (a swap-only subgraph
    // needs no optimizer state at all).
    std::vector<bool> act_used(layers_.size(), false), ckpt_used(blocks_, false);
    for (const Task& t : g_.tasks) {
        if (t.kind == TaskKind::optimizer_update) has_update_ = true;
        const Parsed p = parse_name(t.name);
        if (p.what == "p_c2g" || p.what == "p_s2c") has_weights_ = true;
        if (p.what.rfind("act_", 0) == 0) act_used[4ull * p.block + p.layer] = true;
        if (p.what.rfind("ckpt_", 0) == 0) ckpt_used[p.block] = true;
    }
    const bool need_chunks = has_update_ || has_weights_;
    depths_ = host_ring_depths(g_, opt_);
    ring_ = depths_.states || depths_.params || depths_.weights || depths_.acts;
    acts_on_ssd_ = g_.header.checkpoint_location == "ssd";
    if (ring_ && user_) throw ConfigError("executor: host_ring stages synthetic states only (offsim_execute)");
    h_states_.assign(blocks_, nullptr);
    h_params_.assign(blocks_, nullptr);
    d_grads_.assign(blocks_, nullptr);
    for (std::uint32_t k = 0; k < blocks_ && need_chunks; ++k) {
        if (user_ && (*user_)[k].host_states) {
            h_states_[k] = (*user_)[k].host_states;
            h_params_[k] = (*user_)[k].host_params;
        } else if (!ring_) {
            own_states_.push_back(pin(round_up(state_b)));
            own_params_.push_back(pin(round_up(param_b)));
            h_states_[k] = own_states_.back().p;
            h_params_[k] = own_params_.back().p;
        }
        if (user_ && (*user_)[k].device_grads) {
            d_grads_[k] = (*user_)[k].device_grads;
        } else {
            own_grads_.emplace_back(param_b);
            d_grads_[k] = own_grads_.back().p;
            fill_grads<<<592, 256>>>(static_cast<std::uint16_t*>(own_grads_.back().p), n_, seed + 31 * k);
        }
    }
    // synthetic host states when not provided: generate on the device, copy
    if (need_chunks && !ring_ && !(user_ && (*user_)[0].host_states)) {
        Device tmp(state_b);
        for (std::uint32_t k = 0; k < blocks_; ++k) {
            fill_states<<<592, 256>>>(static_cast<float*>(tmp.p), n_, seed + 7 * k);
            check_cuda(cudaMemcpy(h_states_[k], tmp.p, state_b, cudaMemcpyDeviceToHost), "seed states");
            std::memset(h_params_[k], 0, param_b);
        }
    }
    if (has_update_) {
        const std::uint32_t slots = std::max<std::uint32_t>(2, opt_.state_slots);
        for (std::uint32_t s = 0; s < slots; ++s) slots_.emplace_back(state_b);
    }
    if (has_weights_) {
        std::uint64_t max_w = 0;
        for (const LayerProfile& l : layers_) max_w = std::max(max_w, l.param_bytes);
        wscratch_[0] = Device(max_w);
        wscratch_[1] = Device(max_w);
    }

    // activation / checkpoint units: device originals (pattern), device
    // restore targets, pinned host landing buffers
    act_dev_.resize(layers_.size());
    act_restore_.resize(layers_.size());
    act_host_.resize(layers_.size());
    for (std::size_t i = 0; i < layers_.size(); ++i) {
        if (!swapped_[i] || !act_used[i]) continue;
        const std::uint64_t b = round_up(layers_[i].act_bytes);
        act_dev_[i] = Device(b);
        act_restore_[i] = Device(b);
        if (!(ring_ && acts_on_ssd_)) act_host_[i] = pin(b);
        fill_pattern<<<296, 256>>>(static_cast<std::uint64_t*>(act_dev_[i].p), b / 8, seed ^ (i + 1));
    }
    ckpt_dev_.resize(blocks_);
    ckpt_restore_.resize(blocks_);
    ckpt_host_.resize(blocks_);
    for (std::uint32_t k = 0; k < blocks_; ++k) {
        if (!ckpt_used[k]) continue;
        const std::uint64_t b = round_up(ckpt_bytes_);
        ckpt_dev_[k] = Device(b);
        ckpt_restore_[k] = Device(b);
        if (!(ring_ && acts_on_ssd_)) ckpt_host_[k] = pin(b);
        fill_pattern<<<296, 256>>>(static_cast<std::uint64_t*>(ckpt_dev_[k].p), b / 8,
                                   seed ^ (0xc0ffee00ull + k));
    }
    if (g_.header.variant != ScheduleVariant::overlapped && has_update_)
        for (std::uint32_t k = 0; k < blocks_; ++k) grad_host_.push_back(pin(round_up(param_b)));

    if (ring_) {
        std::uint64_t max_w = 0, max_act = ckpt_bytes_;
        for (std::size_t i = 0; i < layers_.size(); ++i) {
            max_w = std::max(max_w, layers_[i].param_bytes);
            if (swapped_[i]) max_act = std::max(max_act, layers_[i].act_bytes);
        }
        for (std::uint32_t r = 0; r < depths_.states; ++r) state_ring_.push_back(pin(round_up(state_b)));
        for (std::uint32_t r = 0; r < depths_.params; ++r) param_ring_.push_back(pin(round_up(param_b)));
        for (std::uint32_t r = 0; r < depths_.weights; ++r) weight_ring_.push_back(pin(round_up(max_w)));
        for (std::uint32_t r = 0; r < depths_.acts; ++r) act_ring_.push_back(pin(round_up(max_act)));
        assign_ring_slots();
        if (opt_.fixed_buffers) {
            // the rings are every file request's host side: register them
            // once so the kernel does not pin / unpin pages per request
            const auto add = [&](const std::vector<Pinned>& r, std::uint64_t b) {
                for (const Pinned& x : r) io_bufs_.emplace_back(x.p, std::max<std::uint64_t>(b, kAlign));
            };
            add(state_ring_, round_up(state_b));
            add(param_ring_, round_up(param_b));
            add(weight_ring_, round_up(max_w));
            add(act_ring_, round_up(max_act));
            io_registered_ = io_.register_buffers(io_bufs_);
        }
    }

    dataflow_ = opt_.compute_mode == "gemm_dataflow";
    gemm_ = opt_.compute_mode == "gemm" || dataflow_;
    if (!gemm_ && opt_.compute_mode != "spin")
        throw ConfigError("executor: compute_mode must be 'spin', 'gemm' or 'gemm_dataflow'");
    if (dataflow_ && (user_ || !has_update_ || g_.header.variant != ScheduleVariant::overlapped))
        throw ConfigError("executor: gemm_dataflow needs synthetic states, an optimizer and the "
                          "overlapped variant (grads stay in HBM)");
    if (gemm_) {
        const std::uint64_t tokens = model_.batch_size * model_.seq_len;
        const std::uint64_t h = model_.hidden_dim;
        if (tokens > (1ull << 30) || 4 * h > (1ull << 30))
            throw ConfigError("executor: GEMM dimensions out of range");
        // operand extents over fwd (t x in x out), dgrad (t x out -> in) and
        // wgrad (in x t x out): A <= t*4h, B <= max(4h^2, t*4h), C <= max(t*4h, 4h^2)
        const std::uint64_t a_elems = tokens * 4 * h;
        const std::uint64_t bc_elems = std::max(4 * h * h, tokens * 4 * h);
        gemm_a_ = Device(2 * a_elems);
        gemm_b_ = Device(2 * bc_elems);
        gemm_c_ = Device(2 * bc_elems);
        gemm_ws_ = Device(32ull << 20);
        // random bf16 operands (~1e-3): zero operands would understate the
        // tensor cores' power draw and so overstate the rate beside the optimizer
        fill_grads<<<592, 256>>>(static_cast<std::uint16_t*>(gemm_a_.p), a_elems, 3);
        fill_grads<<<592, 256>>>(static_cast<std::uint16_t*>(gemm_b_.p), bc_elems, 4);
        check_cuda(cudaGetLastError(), "fill gemm operands");
        if (cublasCreate(&blas_) != CUBLAS_STATUS_SUCCESS) throw fy::DeviceError("cublasCreate failed");
        cublasSetStream(blas_, lane_stream(ResourceId::gpu_compute));
        cublasSetWorkspace(blas_, gemm_ws_.p, 32ull << 20);
    }
    workspace_ = Device(sizeof(float) * fy::kWorkspaceFloats);
    d_norm_ = Device(sizeof(double));
    d_bad_ = Device(sizeof(int));
    d_mismatch_ = Device(sizeof(unsigned long long));
    check_cuda(cudaMemset(d_norm_.p, 0, sizeof(double)), "memset");
    check_cuda(cudaMemset(d_bad_.p, 0, sizeof(int)), "memset");
    if (dataflow_) {
        // self-check of the grad dataflow: every block's layer j gets the same
        // dW_j = X^T dY (same operands), so the optimizer's accumulated grad
        // sum of squares must equal blocks x sum_j |dW_j * grad_scale|^2
        std::uint64_t max_w = 0;
        for (int j = 0; j < 4; ++j) max_w = std::max<std::uint64_t>(max_w, layers_[j].param_bytes);
        Device scratch(max_w), d_exp(sizeof(double));
        const int tokens = static_cast<int>(model_.batch_size * model_.seq_len);
        cudaStream_t s0 = lane_stream(ResourceId::gpu_compute);
        for (int j = 0; j < 4; ++j) {
            int in = 0, out = 0;
            layer_dims(j, in, out);
            wgrad(s0, tokens, in, out, scratch.p);
            check_cuda(fy::launch_grad_stats(scratch.p, 0, std::uint64_t(in) * out, opt_.adam.grad_scale,
                                             static_cast<double*>(d_exp.p), j > 0,
                                             static_cast<float*>(workspace_.p), nullptr, s0),
                       "expected grad norm");
        }
        double per_block = 0.0;
        check_cuda(cudaStreamSynchronize(s0), "expected grad norm");
        check_cuda(cudaMemcpy(&per_block, d_exp.p, sizeof(double), cudaMemcpyDeviceToHost), "expected grad norm");
        expected_grad_sq_ = per_block * blocks_;
    }
    check_cuda(cudaMemset(d_mismatch_.p, 0, sizeof(unsigned long long)), "memset");

    if (file_tier_) {
        for (const std::string& d : file_dirs()) ::mkdir(d.c_str(), 0700);
        const bool direct = opt_.direct_io && model_.hidden_dim % 64 == 0;
        const std::string stem = "offsim_" + std::to_string(::getpid()) + "_";
        const bool chunks = has_update_ || has_weights_;
        tier_states_bytes_ = chunks ? blocks_ * round_up(state_b) : kAlign;
        f_states_ = std::make_unique<TierFile>(file_dirs(), stem + "states.bin", tier_states_bytes_, direct);
        f_params_ = std::make_unique<TierFile>(file_dirs(), stem + "params.bin",
                                               chunks ? blocks_ * round_up(param_b) : kAlign, direct);
        std::uint64_t off = 0;
        act_file_off_.assign(layers_.size(), 0);
        for (std::size_t i = 0; i < layers_.size(); ++i)
            if (swapped_[i]) {
                act_file_off_[i] = off;
                off += round_up(layers_[i].act_bytes);
            }
        for (std::uint32_t k = 0; k < blocks_; ++k) {
            ckpt_file_off_.push_back(off);
            off += round_up(ckpt_bytes_);
        }
        f_acts_ = std::make_unique<TierFile>(file_dirs(), stem + "acts.bin", std::max<std::uint64_t>(off, kAlign), direct);
        if (!grad_host_.empty())
            f_grads_ = std::make_unique<TierFile>(file_dirs(), stem + "grads.bin", blocks_ * round_up(param_b), direct);
        // the tier holds the initial states / params before the step
        std::unique_ptr<Device> gen;
        Pinned stage_s, stage_p;
        if (ring_ && chunks) {
            gen = std::make_unique<Device>(state_b);
            stage_s = Pinned(round_up(state_b));
            stage_p = Pinned(round_up(param_b));
            std::memset(stage_p.p, 0, round_up(param_b));
        }
        for (std::uint32_t k = 0; k < blocks_ && chunks; ++k) {
            void* src_s = h_states_[k];
            void* src_p = h_params_[k];
            if (ring_) { // generate chunk k on the device, stage it, write it
                fill_states<<<592, 256>>>(static_cast<float*>(gen->p), n_, seed + 7 * k);
                check_cuda(cudaMemcpy(stage_s.p, gen->p, state_b, cudaMemcpyDeviceToHost), "seed states");
                src_s = stage_s.p;
                src_p = stage_p.p;
            }
            IoRequest w{&io_, f_states_->stripe(), src_s, round_up(state_b), k * round_up(state_b), true,
                        false, &io_error_, &io_error_text_, &io_mu_};
            run_io(&w);
            IoRequest wp{&io_, f_params_->stripe(), src_p, round_up(param_b), k * round_up(param_b), true,
                         false, &io_error_, &io_error_text_, &io_mu_};
            run_io(&wp);
        }
        if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
    }
    if (has_update_ && opt_.resident_groups > 0) {
        resident_ = std::min<std::uint32_t>(opt_.resident_groups, blocks_);
        if (opt_.resident_groups == kResidentAuto) {
            // every other buffer of the run is allocated by now; keep room for
            // the calibration's scratch (14 B/param of one group) and a margin
            std::size_t free_b = 0, total_b = 0;
            check_cuda(cudaMemGetInfo(&free_b, &total_b), "meminfo");
            const std::uint64_t keep = 14 * n_ + (1ull << 30) + total_b / 50;
            resident_ = free_b > keep ? static_cast<std::uint32_t>(std::min<std::uint64_t>(
                                            blocks_, (free_b - keep) / state_b))
                                      : 0;
        }
        Pinned tmp;
        for (std::uint32_t k = 0; k < resident_; ++k) {
            res_states_.emplace_back(state_b);
            check_cuda(cudaMemcpy(res_states_.back().p, read_tier_states(k, tmp), state_b, cudaMemcpyHostToDevice),
                       "resident states");
        }
    }
    const AdamHyper& a = opt_.adam;
    scalars_ = fy::make_scalars(a.lr, a.beta1, a.beta2, a.eps, a.weight_decay, a.step,
                                a.adamw_mode, a.bias_correction, a.grad_scale);
    check_cuda(cudaDeviceSynchronize(), "executor setup");
}

MeasuredRates Engine::calibrate() {
    // Burst rates of the engines this run will use (upper bounds for the
    // DES order and the roofline check).
    MeasuredRates r;
    const std::uint64_t bytes = std::min<std::uint64_t>(12 * n_, 512ull << 20);
    Pinned h(bytes);
    cudaEvent_t a, b;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventCreate(&b), "event");
    auto timed = [&](cudaStream_t s, auto&& fn) {
        float best = 1e30f;
        for (int it = 0; it < 3; ++it) {
            check_cuda(cudaEventRecord(a, s), "record");
            fn(s);
            check_cuda(cudaEventRecord(b, s), "record");
            check_cuda(cudaEventSynchronize(b), "sync");
            float ms = 0;
            check_cuda(cudaEventElapsedTime(&ms, a, b), "elapsed");
            best = std::min(best, ms);
        }
        return best * 1e-3;
    };
    Device probe(bytes);
    void* slot = probe.p;
    r.h2d_bps = bytes / timed(lane_stream(ResourceId::link_c2g), [&](cudaStream_t s) {
                    check_cuda(cudaMemcpyAsync(slot, h.p, bytes, cudaMemcpyHostToDevice, s), "h2d");
                });
    r.d2h_bps = bytes / timed(lane_stream(ResourceId::link_g2c), [&](cudaStream_t s) {
                    check_cuda(cudaMemcpyAsync(h.p, slot, bytes, cudaMemcpyDeviceToHost, s), "d2h");
                });
    // Effective link rates: replay this graph's own copy sizes (capped at
    // 256 MiB each, 2 GiB per direction, in task order) per direction, under
    // continuous load from the other direction and alone — small copies and
    // duplex contention included; tier_map blends the two per lane.
    {
        constexpr std::uint64_t kEach = 256ull << 20, kTotal = 2ull << 30;
        std::vector<std::uint64_t> up, down;
        std::uint64_t up_b = 0, down_b = 0, biggest = 0;
        for (const Task& t : g_.tasks) {
            if (t.kind != TaskKind::transfer || t.work <= 0.0) continue;
            const std::uint64_t b = std::min<std::uint64_t>(static_cast<std::uint64_t>(t.work), kEach);
            if (t.resource == ResourceId::link_c2g && up_b < kTotal) { up.push_back(b); up_b += b; }
            if (t.resource == ResourceId::link_g2c && down_b < kTotal) { down.push_back(b); down_b += b; }
            if ((t.resource == ResourceId::link_c2g || t.resource == ResourceId::link_g2c))
                biggest = std::max(biggest, b);
        }
        if (!up.empty() || !down.empty()) {
            Pinned hu(biggest), hd(biggest);
            Device du(biggest), dd(biggest);
            cudaStream_t su = lane_stream(ResourceId::link_c2g), sd = lane_stream(ResourceId::link_g2c);
            cudaEvent_t go, eu, ed;
            check_cuda(cudaEventCreate(&go), "event");
            check_cuda(cudaEventCreate(&eu), "event");
            check_cuda(cudaEventCreate(&ed), "event");
            // each direction's own copies while the OTHER direction is busy
            // the whole time (its copies looped past the measured
            // direction's end): the rate a copy gets when both directions
            // run — small H2D copies under a D2H lose much more than the
            // 1 GiB duplex probe suggests (r02g: a 1.2 MB H2D at 11 GB/s
            // beside a 6 MB D2H)
            auto loaded = [&](cudaStream_t sm, const std::vector<std::uint64_t>& main_sizes, std::uint64_t main_b,
                              bool main_h2d, cudaStream_t so, const std::vector<std::uint64_t>& other_sizes,
                              std::uint64_t other_b) {
                if (main_sizes.empty()) return 0.0;
                if (other_sizes.empty()) return -1.0;  // nothing to contend with
                const int reps = static_cast<int>(std::min<std::uint64_t>(
                    16, 1 + (main_b * 3 / 2 + other_b - 1) / std::max<std::uint64_t>(other_b, 1)));
                double best = 1e30;
                for (int it = 0; it < 2; ++it) {
                    check_cuda(cudaDeviceSynchronize(), "sync");
                    check_cuda(cudaEventRecord(go, so), "record");
                    for (int k = 0; k < reps; ++k)
                        for (const std::uint64_t b : other_sizes)
                            check_cuda(main_h2d ? cudaMemcpyAsync(hd.p, dd.p, b, cudaMemcpyDeviceToHost, so)
                                                : cudaMemcpyAsync(du.p, hu.p, b, cudaMemcpyHostToDevice, so),
                                       "load replay");
                    check_cuda(cudaStreamWaitEvent(sm, go, 0), "wait");
                    check_cuda(cudaEventRecord(ed, sm), "record");
                    for (const std::uint64_t b : main_sizes)
                        check_cuda(main_h2d ? cudaMemcpyAsync(du.p, hu.p, b, cudaMemcpyHostToDevice, sm)
                                            : cudaMemcpyAsync(hd.p, dd.p, b, cudaMemcpyDeviceToHost, sm),
                                   "loaded replay");
                    check_cuda(cudaEventRecord(eu, sm), "record");
                    check_cuda(cudaDeviceSynchronize(), "sync");
                    float ms = 0;
                    check_cuda(cudaEventElapsedTime(&ms, ed, eu), "elapsed");
                    best = std::min(best, ms * 1e-3);
                }
                return main_b / best;
            };
            const double up_loaded = loaded(su, up, up_b, true, sd, down, down_b);
            const double down_loaded = loaded(sd, down, down_b, false, su, up, up_b);
            // the same copies one direction at a time
            auto simplex = [&](cudaStream_t st, const std::vector<std::uint64_t>& sizes, bool h2d) {
                double best = 1e30;
                for (int it = 0; it < 2 && !sizes.empty(); ++it) {
                    check_cuda(cudaDeviceSynchronize(), "sync");
                    check_cuda(cudaEventRecord(go, st), "record");
                    for (const std::uint64_t b : sizes)
                        check_cuda(h2d ? cudaMemcpyAsync(du.p, hu.p, b, cudaMemcpyHostToDevice, st)
                                       : cudaMemcpyAsync(hd.p, dd.p, b, cudaMemcpyDeviceToHost, st),
                                   "simplex replay");
                    check_cuda(cudaEventRecord(eu, st), "record");
                    check_cuda(cudaEventSynchronize(eu), "sync");
                    float ms = 0;
                    check_cuda(cudaEventElapsedTime(&ms, go, eu), "elapsed");
                    best = std::min(best, ms * 1e-3);
                }
                return best;
            };
            if (up_b > 0) r.h2d_simplex_effective_bps = up_b / simplex(su, up, true);
            if (down_b > 0) r.d2h_simplex_effective_bps = down_b / simplex(sd, down, false);
            // no copies the other way: the loaded rate is the simplex one
            r.h2d_effective_bps = up_loaded < 0 ? r.h2d_simplex_effective_bps : up_loaded;
            r.d2h_effective_bps = down_loaded < 0 ? r.d2h_simplex_effective_bps : down_loaded;
            cudaEventDestroy(go);
            cudaEventDestroy(eu);
            cudaEventDestroy(ed);
        }
    }
    // fused kernel rate on a scratch copy (does not touch the real states)
    r.optimizer_params_per_s = 1e12; // no optimizer task: the lane stays empty
    if (has_update_) {
        Device st(12 * n_), gr(2 * n_);
        fill_states<<<592, 256>>>(static_cast<float*>(st.p), n_, 1);
        fill_grads<<<592, 256>>>(static_cast<std::uint16_t*>(gr.p), n_, 2);
        fy::AdamLaunch l{};
        l.master = static_cast<float*>(st.p);
        l.m = l.master + n_;
        l.v = l.master + 2 * n_;
        l.grad = gr.p;
        l.grad_dtype = 0;
        l.param = gr.p;
        l.param_dtype = 0;
        l.n = n_;
        l.s = scalars_;
        const double sec = timed(lane_stream(ResourceId::cpu_compute), [&](cudaStream_t s) {
            check_cuda(fy::launch_adamw(l, s), "calibrate adamw");
        });
        r.optimizer_params_per_s = n_ / sec;
    }
    if (file_tier_) {
        // Best of three, writes unsynced exactly as the executor issues them:
        // the rates must be upper bounds for the roofline check. Requests of
        // a few MB (smaller than the calibration size) can see device-cache
        // speedups, hence the extra IO headroom applied in b200_hardware.
        // a scratch file in the same directory: the tier files already hold
        // the initial states and must not be touched by the probe
        const bool direct = opt_.direct_io && model_.hidden_dim % 64 == 0;
        TierFile probe_file(file_dirs(), "offsim_" + std::to_string(::getpid()) + "_probe.bin",
                            round_up(bytes), direct);
        // the probe buffer joins the registration while it is in use, so the
        // calibrated rates are those of the requests the iteration issues
        if (io_registered_) {
            auto with_probe = io_bufs_;
            with_probe.emplace_back(h.p, round_up(bytes));
            io_registered_ = io_.register_buffers(with_probe) ? io_registered_ : 0;
        }
        // back to the rings alone before the probe buffer is freed (a stale
        // registration would alias whatever is mapped there next)
        struct Reregister {
            Engine* e;
            ~Reregister() {
                if (e->io_registered_) e->io_registered_ = e->io_.register_buffers(e->io_bufs_);
            }
        } reregister{this};
        IoRequest w{&io_, probe_file.stripe(), h.p, round_up(bytes), 0, true, false, &io_error_,
                    &io_error_text_, &io_mu_};
        IoRequest rd = w;
        rd.write = false;
        double best_w = 1e30, best_r = 1e30;
        for (int it = 0; it < 3; ++it) {
            const auto t0 = std::chrono::steady_clock::now();
            run_io(&w);
            const auto t1 = std::chrono::steady_clock::now();
            run_io(&rd);
            const auto t2 = std::chrono::steady_clock::now();
            best_w = std::min(best_w, std::chrono::duration<double>(t1 - t0).count());
            best_r = std::min(best_r, std::chrono::duration<double>(t2 - t1).count());
        }
        r.file_write_bps = bytes / best_w;
        r.file_read_bps = bytes / best_r;
        // effective: replay the graph's own file-lane requests in task
        // order (<= 4 GiB of reads and <= 4 GiB of writes per pass, so a
        // write-heavy prefix cannot leave the reads unsampled) through the
        // iteration's own host buffers
        // and file extents (FileOp), so the replay meets the same
        // buffer / extent state and the same request mix as the iteration
        // (r02at: a replay through the probe buffer read ~5.5 GB/s where the
        // iteration's reads into its per-checkpoint buffers got ~3 on the
        // same virtio disk). Writes into the state / param files go to the
        // probe file instead (the tier holds the initial states); every
        // other request leaves no trace: reads return what the buffers
        // already hold or what the iteration overwrites before use, and
        // the activation / gradient extents are rewritten by the iteration
        // before they are read. With warm_files two passes, the second one
        // timed: the lane as every iteration after the first finds it.
        constexpr std::uint64_t kReplay = 8ull << 30, kPerDir = 4ull << 30;
        struct Pass {
            double rd_b = 0, rd_s = 0, wr_b = 0, wr_s = 0;
        };
        auto replay = [&]() {
            Pass p;
            std::uint64_t wcur = round_up(bytes);
            for (const Task& t : g_.tasks) {
                FileOp fo;
                if (!file_op(t, fo)) continue;
                if (p.rd_b >= double(kPerDir) && p.wr_b >= double(kPerDir)) break;
                if ((fo.write ? p.wr_b : p.rd_b) >= double(kPerDir)) continue;
                IoRequest op{&io_, fo.file->stripe(), fo.buf, round_up(fo.bytes), fo.offset, fo.write, false,
                             &io_error_, &io_error_text_, &io_mu_};
                if (fo.write && (fo.file == f_states_.get() || fo.file == f_params_.get())) {
                    if (wcur + op.bytes > kReplay) wcur = 0;
                    op.file = probe_file.stripe();
                    op.offset = wcur;
                    wcur += op.bytes;
                }
                const auto t0 = std::chrono::steady_clock::now();
                run_io(&op);
                const double sec =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                (op.write ? p.wr_b : p.rd_b) += static_cast<double>(op.bytes);
                (op.write ? p.wr_s : p.rd_s) += sec;
            }
            return p;
        };
        Pass alone;
        for (int pass = 0; pass < (opt_.warm_files ? 2 : 1); ++pass) alone = replay();
        if (alone.rd_s > 0) r.file_read_effective_bps = alone.rd_b / alone.rd_s;
        if (alone.wr_s > 0) r.file_write_effective_bps = alone.wr_b / alone.wr_s;
        // the same replay while both copy engines stream pinned host memory
        // the whole time: GPU DMA into host memory slows the file lane (on
        // the leases' virtio disk by ~22%, profiles/r02bc_file_rw_link_load.txt);
        // tier_map blends the two by the share of the file lane's planned
        // busy time a link lane overlaps (MeasuredRates::ssd_link_overlap)
        bool has_link = false;
        for (const Task& t : g_.tasks)
            has_link |= t.work > 0.0 && (t.resource == ResourceId::link_c2g || t.resource == ResourceId::link_g2c);
        const double t_alone = alone.rd_s + alone.wr_s;
        if (has_link && t_alone > 0) {
            constexpr std::uint64_t kCopy = 256ull << 20;
            Pinned lh(kCopy), ld(kCopy);
            Device du(kCopy), dd(kCopy);
            const double rate = std::max(r.h2d_bps, r.d2h_bps) > 0 ? std::max(r.h2d_bps, r.d2h_bps) : 55e9;
            const int copies = static_cast<int>(std::min(20000.0, std::ceil(1.5 * t_alone * rate / kCopy) + 2));
            cudaStream_t su = lane_stream(ResourceId::link_c2g), sd = lane_stream(ResourceId::link_g2c);
            for (int c = 0; c < copies; ++c) {
                check_cuda(cudaMemcpyAsync(du.p, lh.p, kCopy, cudaMemcpyHostToDevice, su), "load H2D");
                check_cuda(cudaMemcpyAsync(ld.p, dd.p, kCopy, cudaMemcpyDeviceToHost, sd), "load D2H");
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(5));  // both engines running
            const Pass loaded = replay();
            check_cuda(cudaStreamSynchronize(su), "load H2D");
            check_cuda(cudaStreamSynchronize(sd), "load D2H");
            if (loaded.rd_s > 0) r.file_read_loaded_bps = loaded.rd_b / loaded.rd_s;
            if (loaded.wr_s > 0) r.file_write_loaded_bps = loaded.wr_b / loaded.wr_s;
        }
        if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
    }
    r.compute_flops = opt_.compute_rate > 0 ? opt_.compute_rate : 0.0;
    if (gemm_) {
        // the largest layer GEMM of the model, best of three
        const int tokens = static_cast<int>(model_.batch_size * model_.seq_len);
        const int h = static_cast<int>(model_.hidden_dim);
        const double sec = timed(lane_stream(ResourceId::gpu_compute),
                                 [&](cudaStream_t s) { gemm(s, tokens, 4 * h, h); });
        r.compute_headroom = 1.05;
        r.compute_flops = 2.0 * tokens * 4.0 * h * h / sec * r.compute_headroom;  // upper bound
    }
    // effective compute rate: the graph's own compute tasks (up to ~0.25 s
    // of nominal work, in task order) replayed back to back on the compute
    // lane, each bracketed by timing events exactly as the run brackets it —
    // per-kernel launch / event overhead and small-GEMM efficiency included
    if (r.compute_flops > 0) {
        compute_rate_ = r.compute_flops;
        cudaStream_t s = lane_stream(ResourceId::gpu_compute);
        std::vector<const Task*> replay;
        double nominal = 0, work = 0;
        for (const Task& t : g_.tasks) {
            if (t.kind != TaskKind::compute || t.work <= 0.0) continue;
            replay.push_back(&t);
            work += t.work;
            nominal += t.work / r.compute_flops;
            if (nominal > 0.25) break;
        }
        double best = 1e30;
        for (int it = 0; it < 2 && !replay.empty(); ++it) {
            check_cuda(cudaDeviceSynchronize(), "sync");
            for (const Task* t : replay) {
                check_cuda(cudaEventRecord(events_[2 * t->id], s), "record");
                issue_compute(*t, parse_name(t->name), s, true);
                check_cuda(cudaEventRecord(events_[2 * t->id + 1], s), "record");
            }
            check_cuda(cudaDeviceSynchronize(), "compute replay");
            double sum = 0;
            for (const Task* t : replay) {
                float ms = 0;
                check_cuda(cudaEventElapsedTime(&ms, events_[2 * t->id], events_[2 * t->id + 1]), "elapsed");
                sum += ms * 1e-3;
            }
            best = std::min(best, sum);
        }
        if (!replay.empty() && best > 0) r.compute_effective_flops = work / best;
    }
    std::size_t free_b = 0, total_b = 0;
    check_cuda(cudaMemGetInfo(&free_b, &total_b), "meminfo");
    r.gpu_mem = total_b;
    r.cpu_mem = static_cast<std::uint64_t>(::sysconf(_SC_PHYS_PAGES)) *
                static_cast<std::uint64_t>(::sysconf(_SC_PAGESIZE));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return r;
}

// Ring slot of every task that touches a staging ring; same use order as
// add_host_ring_edges (task id order), so the graph's reuse edges protect
// exactly these slots.
void Engine::assign_ring_slots() {
    std::map<std::string, std::uint32_t> id_of;
    for (const Task& t : g_.tasks) id_of[t.name] = t.id;
    std::uint32_t ns = 0, np = 0, nw = 0, na = 0;
    auto tie = [&](const std::string& name, int slot) {
        const auto it = id_of.find(name);
        if (it != id_of.end()) ring_slot_[it->second] = slot;
    };
    auto swap_name = [](std::string n, const char* a, const char* b) {
        n.replace(n.find(a), std::strlen(a), b);
        return n;
    };
    for (const Task& t : g_.tasks) {
        const std::string& n = t.name;
        if (n.rfind("opt state_s2c ", 0) == 0) {
            const int slot = static_cast<int>(ns++ % depths_.states);
            for (const char* w : {"state_s2c", "state_h2d", "state_d2h", "state_c2s"})
                tie(swap_name(n, "state_s2c", w), slot);
        } else if (n.rfind("opt param_d2h ", 0) == 0) {
            const int slot = static_cast<int>(np++ % depths_.params);
            tie(n, slot);
            tie(swap_name(n, "param_d2h", "param_c2s"), slot);
        } else if (n.find(" p_s2c ") != std::string::npos) {
            const int slot = static_cast<int>(nw++ % depths_.weights);
            tie(n, slot);
            tie(swap_name(n, "p_s2c", "p_c2g"), slot);
        } else if (acts_on_ssd_ && (n.rfind("fwd act_g2c ", 0) == 0 || n.rfind("fwd ckpt_g2c ", 0) == 0)) {
            const int slot = static_cast<int>(na++ % depths_.acts);
            tie(n, slot);
            tie(swap_name(n, "_g2c", "_c2s"), slot);
        } else if (acts_on_ssd_ && (n.rfind("bwd act_s2c ", 0) == 0 || n.rfind("bwd ckpt_s2c ", 0) == 0)) {
            const int slot = static_cast<int>(na++ % depths_.acts);
            tie(n, slot);
            tie(swap_name(n, "_s2c", "_c2g"), slot);
        }
    }
}

// Initial [master|m|v] of chunk k from its tier: the pinned host copy, or
// (file tier with staging rings) a read of its file region into `tmp`.
void* Engine::read_tier_states(std::uint32_t k, Pinned& tmp) {
    const std::uint64_t state_b = 12 * n_;
    if (h_states_[k]) return h_states_[k];  // the host copy the tier was seeded from
    if (!tmp.p) tmp = Pinned(round_up(state_b));
    IoRequest r{&io_, f_states_->stripe(), tmp.p, round_up(state_b), k * round_up(state_b), false, false,
                &io_error_, &io_error_text_, &io_mu_};
    run_io(&r);
    if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
    return tmp.p;
}

// Resident groups' final states go back to their tier after the run (host
// copy and/or file region), so checksums and caller buffers see them.
void Engine::write_back_resident() {
    const std::uint64_t state_b = 12 * n_;
    Pinned tmp;
    for (std::uint32_t k = 0; k < resident_; ++k) {
        void* dst = h_states_[k];
        if (!dst) {
            if (!tmp.p) tmp = Pinned(round_up(state_b));
            dst = tmp.p;
        }
        check_cuda(cudaMemcpy(dst, res_states_[k].p, state_b, cudaMemcpyDeviceToHost), "resident write-back");
        if (file_tier_) {
            IoRequest w{&io_, f_states_->stripe(), dst, round_up(state_b), k * round_up(state_b), true, false,
                        &io_error_, &io_error_text_, &io_mu_};
            run_io(&w);
        }
    }
    if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
}

// FNV-1a over 64-bit words of every chunk's final [master|m|v], read back
// from the file tier (or the pinned host copies) after the run.
std::uint64_t Engine::checksum_states() {
    const std::uint64_t state_b = 12 * n_;
    std::uint64_t h = 1469598103934665603ull;
    Pinned tmp;
    if (file_tier_) tmp = Pinned(round_up(state_b));
    for (std::uint32_t k = 0; k < blocks_; ++k) {
        const void* src = h_states_[k];
        if (file_tier_) {
            IoRequest r{&io_, f_states_->stripe(), tmp.p, round_up(state_b), k * round_up(state_b), false, false,
                        &io_error_, &io_error_text_, &io_mu_};
            run_io(&r);
            src = tmp.p;
        }
        if (!src) continue;
        const auto* w = static_cast<const std::uint64_t*>(src);
        for (std::uint64_t i = 0; i < state_b / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
    }
    if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
    return h;
}

// C[m x n] = A[m x k] * B[k x n], bf16 in / bf16 out, fp32 accumulate
// (row-major operands expressed as column-major transposes for cuBLAS).
void Engine::gemm(cudaStream_t s, int m, int n, int k) {
    cublasSetStream(blas_, s);
    const float alpha = 1.0f, beta = 0.0f;
    const cublasStatus_t st = cublasGemmEx(blas_, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &alpha, gemm_b_.p,
                                           CUDA_R_16BF, n, gemm_a_.p, CUDA_R_16BF, k, &beta, gemm_c_.p,
                                           CUDA_R_16BF, n, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) throw fy::DeviceError("cublasGemmEx failed: status " + std::to_string(st));
}

void Engine::wgrad(cudaStream_t s, int tokens, int in, int out, void* dst) {
    // row-major dW[in x out] = X[t x in]^T * dY[t x out]; in cuBLAS's
    // column-major view: dW_cm[out x in] = dY_cm[out x t] * (X_cm[in x t])^T
    cublasSetStream(blas_, s);
    const float alpha = 1.0f, beta = 0.0f;
    const cublasStatus_t st = cublasGemmEx(blas_, CUBLAS_OP_N, CUBLAS_OP_T, out, in, tokens, &alpha, gemm_b_.p,
                                           CUDA_R_16BF, out, gemm_a_.p, CUDA_R_16BF, in, &beta, dst,
                                           CUDA_R_16BF, out, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) throw fy::DeviceError("cublasGemmEx (wgrad) failed: status " + std::to_string(st));
}

// One compute task: the layer's real bf16 GEMMs (gemm modes; attention
// extras as a timed spin) or a kernel that spins for work / compute_rate_.
// replay (calibration): gradients are not written (wgrad into scratch).
void Engine::issue_compute(const Task& t, const Parsed& p, cudaStream_t s, bool replay) {
    const std::uint32_t k = p.block;
    const int j = p.layer;
    if (gemm_) {
        int in = 0, out = 0;
        layer_dims(j, in, out);
        const int tokens = static_cast<int>(model_.batch_size * model_.seq_len);
        const bool bwd = p.phase == "bwd" && p.what == "compute";
        if (bwd) {
            gemm(s, tokens, in, out);  // dgrad: dY[t x out] * W^T -> dX[t x in]
            if (dataflow_ && !replay)  // wgrad straight into the block's grad buffer (the optimizer's input)
                wgrad(s, tokens, in, out, static_cast<char*>(const_cast<void*>(d_grads_[k])) + layer_offset(j));
            else
                gemm(s, in, out, tokens);  // wgrad: X^T[in x t] * dY -> dW[in x out]
        } else {
            gemm(s, tokens, out, in);  // forward / recompute
        }
        // attention-score extras (extra_flops_per_block) stay timed
        const double extra = t.work - (bwd ? 4.0 : 2.0) * double(tokens) * in * out;
        if (extra > 1.0) spin_kernel<<<1, 32, 0, s>>>(static_cast<std::uint64_t>(extra / compute_rate_ * 1e9));
    } else {
        spin_kernel<<<1, 32, 0, s>>>(static_cast<std::uint64_t>(t.work / compute_rate_ * 1e9));
    }
    check_cuda(cudaGetLastError(), "compute launch");
}

bool Engine::file_op(const Task& t, FileOp& op) {
    if (t.resource != ResourceId::link_ssd || t.work <= 0.0) return false;
    const Parsed p = parse_name(t.name);
    const std::uint32_t k = p.block;
    const int j = p.layer;
    const std::uint64_t li = j >= 0 ? 4ull * k + j : 0;
    const std::uint64_t state_b = 12 * n_, param_b = 2 * n_;
    const std::string& w = p.what;
    if (w == "state_s2c" || w == "state_c2s") {
        op = {f_states_.get(), host_states(t.id, k), state_b, k * round_up(state_b), w == "state_c2s", false};
    } else if (w == "param_c2s") {
        op = {f_params_.get(), host_params(t.id, k), param_b, k * round_up(param_b), true, false};
    } else if (w == "p_s2c") {
        const std::uint64_t off = layer_offset(j);
        op = {f_params_.get(), host_weights(t.id, k, off), layers_[li].param_bytes, k * round_up(param_b) + off,
              false, false};
    } else if (w == "act_c2s" || w == "act_s2c") {
        const bool wr = w == "act_c2s";
        op = {f_acts_.get(), host_act(t.id, act_host_[li]), layers_[li].act_bytes, act_file_off_[li], wr,
              wr && opt_.verify_swaps};
    } else if (w == "ckpt_c2s" || w == "ckpt_s2c") {
        const bool wr = w == "ckpt_c2s";
        op = {f_acts_.get(), host_act(t.id, ckpt_host_[k]), ckpt_bytes_, ckpt_file_off_[k], wr,
              wr && opt_.verify_swaps};
    } else if (w == "grad_c2s" || w == "grad_s2c") {
        op = {f_grads_.get(), grad_host_[k].p, param_b, k * round_up(param_b), w == "grad_c2s", false};
    } else {
        return false;
    }
    if (!op.file) throw InvariantError("executor: no tier file for task '" + t.name + "'");
    return true;
}

// Untimed, before calibration: the file lane as every iteration after the
// first finds it (ExecOptions::warm_files). (1) Every extent the iteration
// WRITES in the activation / checkpoint / gradient files is written once
// (setup already wrote the state and param files); (2) every host buffer a
// file READ lands in receives one read (of its own extent). On the leases'
// virtio disk the first write to a new extent runs at ~3.6-3.9 GB/s against
// ~5 GB/s for an overwrite, and the first device DMA into a host region at
// ~2.8 GB/s against ~4.6 (profiles/r02aq_file_rw_*.txt) — one cold
// iteration measured first-touch costs, not the lane. Contents: the writes
// only allocate extents that the iteration overwrites before reading them;
// state / param reads return the bytes those buffers already hold (the
// tier files were written from them at setup), and activation / gradient
// buffers are overwritten by their D2H before any use.
double Engine::warm_file_lane() {
    if (!file_tier_ || !opt_.warm_files) return 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    std::set<std::pair<const void*, std::uint64_t>> written, read;
    for (int pass = 0; pass < 2; ++pass) {
        for (const Task& t : g_.tasks) {
            FileOp op;
            if (!file_op(t, op) || op.write != (pass == 0)) continue;
            if (op.write && op.file != f_acts_.get() && op.file != f_grads_.get()) continue;
            auto& seen = op.write ? written : read;
            // writes: every extent once; reads: every host buffer once
            if (!seen.emplace(op.write ? static_cast<const void*>(op.file) : op.buf, op.write ? op.offset : 0)
                     .second)
                continue;
            IoRequest r{&io_, op.file->stripe(), op.buf, round_up(op.bytes), op.offset, op.write, false,
                        &io_error_, &io_error_text_, &io_mu_};
            run_io(&r);
        }
    }
    if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::issue(const Task& t, ExecReport& rep) {
    cudaStream_t s = lane_stream(t.resource);
    for (const std::uint32_t d : t.deps)
        if (g_.tasks[d].resource != t.resource)
            check_cuda(cudaStreamWaitEvent(s, end_dep(d), 0), "wait dep");
    const Parsed p = parse_name(t.name);
    const std::uint32_t k = p.block;
    const int j = p.layer;
    const std::uint64_t li = j >= 0 ? 4ull * k + j : 0;
    auto phys = [&](const char* engine, std::uint64_t bytes) {
        rep.physical_bytes[std::string(engine) + "/" + to_string(t.payload)] += static_cast<double>(bytes);
    };
    auto h2d = [&](void* dst, const void* src, std::uint64_t bytes) {
        check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
        phys("h2d", bytes);
    };
    auto d2h = [&](void* dst, const void* src, std::uint64_t bytes) {
        check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
        phys("d2h", bytes);
    };
    auto file = [&](const TierFile& f, void* buf, std::uint64_t bytes, std::uint64_t off, bool write,
                    bool poison) {
        io_reqs_.push_back(std::make_unique<IoRequest>(IoRequest{&io_, f.stripe(), buf, round_up(bytes), off, write,
                                                            poison, &io_error_, &io_error_text_, &io_mu_}));
        check_cuda(cudaLaunchHostFunc(s, run_io, io_reqs_.back().get()), "host io");
        phys(write ? "file_write" : "file_read", bytes);
    };

    // Instrumentation is one timing event per task, at its END: a task
    // starts when its lane's previous task and its dependencies are done, so
    // its start is reconstructed from those ends after the run (run()). A
    // start event-record node per task cost ~5-9 us of device latency on
    // every edge of the critical path (r02f: C1 with HBM-resident states
    // spent ~19 us per compute task in them).
    issued_.push_back(t.id);
    const std::uint64_t state_b = 12 * n_, param_b = 2 * n_;
    const std::string& w = p.what;
    if (t.work <= 0.0) {
        // zero-byte task of the mapped graph (host tier SSD hop, HBM grads):
        // its dependencies are waited on above (the lane stays FIFO behind
        // them) and its end is a dependency point only — no GPU node
        check_cuda(cudaEventRecord(deps_[t.id], s), "record dep");
        return;
    } else if (t.kind == TaskKind::compute) {
        issue_compute(t, p, s, false);
        if (!gemm_) ++rep.kernel_launches;  // cuBLAS GEMMs are not ours
    } else if (t.kind == TaskKind::optimizer_update) {
        const int slot = slot_of(k);
        fy::AdamLaunch l{};
        l.master = static_cast<float*>(is_resident(k) ? res_states_[k].p : slots_[slot].p);
        l.m = l.master + n_;
        l.v = l.master + 2 * n_;
        l.grad = d_grads_[k];
        l.grad_dtype = 0;
        l.param = const_cast<void*>(d_grads_[k]); // grad buffer becomes the params
        l.param_dtype = 0;
        l.n = n_;
        l.s = scalars_;
        l.grad_sq_sum = static_cast<double*>(d_norm_.p);
        l.accumulate_sq = 1;
        l.workspace = static_cast<float*>(workspace_.p);
        l.nonfinite = static_cast<int*>(d_bad_.p);
        check_cuda(fy::launch_adamw(l, s), "opt update");
        rep.kernel_launches += 2;
    } else if (w == "state_h2d") {
        // the slot's previous user (state_d2h of group m - slots) is a dep
        h2d(slots_[slot_of(k)].p, host_states(t.id, k), state_b);
    } else if (w == "state_d2h") {
        d2h(host_states(t.id, k), slots_[slot_of(k)].p, state_b);
    } else if (w == "param_d2h") {
        d2h(host_params(t.id, k), d_grads_[k], param_b);
    } else if (FileOp op; file_op(t, op)) {
        file(*op.file, op.buf, op.bytes, op.offset, op.write, op.poison);
    } else if (w == "p_c2g") {
        void* dst = wscratch_[wscratch_turn_ ^= 1].p;
        h2d(dst, host_weights(t.id, k, layer_offset(j)), layers_[li].param_bytes);
    } else if (w == "act_g2c") {
        d2h(host_act(t.id, act_host_[li]), act_dev_[li].p, layers_[li].act_bytes);
    } else if (w == "act_c2g") {
        h2d(act_restore_[li].p, host_act(t.id, act_host_[li]), layers_[li].act_bytes);
    } else if (w == "ckpt_g2c") {
        d2h(host_act(t.id, ckpt_host_[k]), ckpt_dev_[k].p, ckpt_bytes_);
    } else if (w == "ckpt_c2g") {
        h2d(ckpt_restore_[k].p, host_act(t.id, ckpt_host_[k]), ckpt_bytes_);
    } else if (w == "grad_g2c") {
        d2h(grad_host_[k].p, d_grads_[k], param_b);
    } else if (w == "grad_h2d") {
        h2d(const_cast<void*>(d_grads_[k]), grad_host_[k].p, param_b);
    } else {
        throw InvariantError("executor: no operation for task '" + t.name + "'");
    }
    record_time(events_[2 * t.id + 1], s);
    if (capturing_) check_cuda(cudaEventRecord(deps_[t.id], s), "record dep");
}

// Graph mode: the whole iteration captured once into ONE CUDA graph (lane
// streams forked from / joined into streams_[0]; cross-lane dependencies are
// graph edges; each task's start / end are event-record nodes), instantiated
// before the timed region and launched as one unit. The GPU then resolves
// every dependency itself: no host issue latency between tasks (stream mode
// issues ~5 API calls per task from one host thread, which bounds small
// iterations — C1 with HBM-resident states was host-issue bound, r02d).
bool Engine::run_graph(const std::vector<std::pair<std::uint64_t, std::uint32_t>>& order, ExecReport& rep) {
    const ExecReport saved = rep;
    const std::size_t io_mark = io_reqs_.size();
    const int turn = wscratch_turn_;
    cudaStream_t origin = streams_[0];
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t fork = nullptr;
    bool ok = false;
    try {
        check_cuda(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event");
        check_cuda(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed), "begin capture");
        capturing_ = true;
        record_time(base_, origin);
        check_cuda(cudaEventRecord(fork, origin), "fork");
        for (int r = 1; r < 5; ++r) check_cuda(cudaStreamWaitEvent(streams_[r], fork, 0), "fork wait");
        for (const auto& [start, id] : order) issue(g_.tasks[id], rep);
        for (int r = 1; r < 5; ++r) {  // join every lane back into the origin
            check_cuda(cudaEventRecord(fork, streams_[r]), "join");
            check_cuda(cudaStreamWaitEvent(origin, fork, 0), "join wait");
        }
        capturing_ = false;
        check_cuda(cudaStreamEndCapture(origin, &graph), "end capture");
        check_cuda(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
        check_cuda(cudaGraphUpload(exec, origin), "graph upload");
        check_cuda(cudaStreamSynchronize(origin), "graph upload sync");
        check_cuda(cudaGraphLaunch(exec, origin), "graph launch");
        check_cuda(cudaStreamSynchronize(origin), "graph run");
        ok = true;
    } catch (const std::exception&) {
        if (capturing_) {  // abandon the capture; the stream leaves capture mode
            capturing_ = false;
            cudaGraph_t partial = nullptr;
            cudaStreamEndCapture(origin, &partial);
            if (partial) cudaGraphDestroy(partial);
        }
        cudaGetLastError();
        if (exec) {  // failed while running: a real device error, not a capture limit
            cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
            if (fork) cudaEventDestroy(fork);
            throw;
        }
        rep = saved;  // the stream-mode issue starts from a clean report
        issued_.clear();
        io_reqs_.resize(io_mark);
        wscratch_turn_ = turn;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (fork) cudaEventDestroy(fork);
    return ok;
}

void Engine::run(const SimTrace& planned, ExecReport& rep) {
    compute_rate_ = rep.hw_exec.gpu_tput;
    // issue order = planned start order (ties: task id, always topological)
    std::vector<std::pair<std::uint64_t, std::uint32_t>> order;
    order.reserve(planned.events.size());
    for (const TraceEvent& e : planned.events) order.emplace_back(e.start_ns, e.task_id);
    std::sort(order.begin(), order.end());

    check_cuda(cudaDeviceSynchronize(), "pre-run sync");
    issued_.clear();
    rep.launch_mode = "stream";
    if (opt_.launch == "graph" && run_graph(order, rep)) {
        rep.launch_mode = "graph";
    } else {
        check_cuda(cudaEventRecord(base_, streams_[0]), "base");
        for (int r = 1; r < 5; ++r) check_cuda(cudaStreamWaitEvent(streams_[r], base_, 0), "base wait");
        for (const auto& [start, id] : order) issue(g_.tasks[id], rep);
    }
    check_cuda(cudaDeviceSynchronize(), "executor run");
    (void)g_io_done.load(std::memory_order_acquire);  // pairs with run_io's release
    if (io_error_) throw InfeasibleError("file tier: " + io_error_text_);

    // swap integrity: every restored buffer equals its original
    if (opt_.verify_swaps) {
        auto cmp = [&](const Device& a, const Device& b, std::uint64_t bytes) {
            count_mismatch<<<296, 256>>>(static_cast<const std::uint64_t*>(a.p),
                                        static_cast<const std::uint64_t*>(b.p), bytes / 8,
                                        static_cast<unsigned long long*>(d_mismatch_.p));
            ++rep.swap_checks;
        };
        for (const Task& t : g_.tasks) {
            if (t.work <= 0.0) continue;
            const Parsed p = parse_name(t.name);
            if (p.what == "act_c2g") cmp(act_dev_[4ull * p.block + p.layer], act_restore_[4ull * p.block + p.layer],
                                         layers_[4ull * p.block + p.layer].act_bytes / 8 * 8);
            if (p.what == "ckpt_c2g") cmp(ckpt_dev_[p.block], ckpt_restore_[p.block], ckpt_bytes_ / 8 * 8);
        }
        unsigned long long bad = 0;
        check_cuda(cudaMemcpy(&bad, d_mismatch_.p, sizeof bad, cudaMemcpyDeviceToHost), "mismatch");
        rep.swap_mismatches = bad;
    }
    check_cuda(cudaMemcpy(&rep.grad_sq_sum, d_norm_.p, sizeof(double), cudaMemcpyDeviceToHost), "norm");
    rep.expected_grad_sq_sum = dataflow_ ? expected_grad_sq_ : -1.0;
    rep.pinned_host_bytes = pinned_bytes_;
    // the iteration's file requests (the write-back / checksum reads below
    // use scratch buffers outside the registration)
    rep.io_fixed_requests = io_.fixed_requests();
    rep.io_plain_requests = io_.plain_requests();
    if (resident_ > 0) write_back_resident();
    if (opt_.checksum_states && has_update_) rep.state_checksum = checksum_states();
    check_cuda(cudaMemcpy(&rep.nonfinite, d_bad_.p, sizeof(int), cudaMemcpyDeviceToHost), "flag");

    // real trace: measured ends (timing events); each start = the later of
    // its lane predecessor's end and its dependencies' ends (when the stream
    // let the operation begin); zero-work tasks take no time
    SimTrace& tr = rep.trace;
    tr.header = g_.header;
    tr.events.clear();
    std::vector<std::uint64_t> end_ns(g_.tasks.size(), 0);
    std::map<ResourceId, std::uint64_t> lane_end;
    std::vector<TraceEvent> evs(g_.tasks.size());
    for (const std::uint32_t id : issued_) {
        const Task& t = g_.tasks[id];
        std::uint64_t start = lane_end[t.resource];
        for (const std::uint32_t d : t.deps) start = std::max(start, end_ns[d]);
        std::uint64_t end = start;
        if (t.work > 0.0) {
            float ms1 = 0;
            check_cuda(cudaEventElapsedTime(&ms1, base_, events_[2 * t.id + 1]), "elapsed");
            end = static_cast<std::uint64_t>(std::llround(std::max(0.0f, ms1) * 1e6));
            if (end < start) start = end;  // timer jitter: never a negative duration
        }
        end_ns[id] = end;
        lane_end[t.resource] = end;
        evs[id] = TraceEvent{t.id, t.resource, t.dir, t.payload, t.work, start, end};
    }
    for (const Task& t : g_.tasks) {
        const TraceEvent& e = evs[t.id];
        tr.events.push_back(e);
        tr.makespan_ns = std::max(tr.makespan_ns, e.end_ns);
        tr.busy_ns[t.resource] += e.end_ns - e.start_ns;
    }
    std::sort(tr.events.begin(), tr.events.end(), [](const TraceEvent& a, const TraceEvent& b) {
        return a.end_ns != b.end_ns ? a.end_ns < b.end_ns : a.task_id < b.task_id;
    });
    // peak memory by replaying the effects over the real timeline
    std::vector<std::tuple<std::uint64_t, int, std::uint32_t>> edges;
    for (const TraceEvent& e : tr.events) {
        edges.emplace_back(e.start_ns, 1, e.task_id);
        edges.emplace_back(e.end_ns, 0, e.task_id);
    }
    std::sort(edges.begin(), edges.end());
    std::map<ResourceId, std::int64_t> level = g_.initial_mem;
    tr.peak_mem = level;
    for (const auto& [time, is_start, id] : edges) {
        for (const MemEffect& fx : g_.tasks[id].mem_effects) {
            if (fx.at_start != (is_start == 1)) continue;
            level[fx.mem] += fx.delta_bytes;
            tr.peak_mem[fx.mem] = std::max(tr.peak_mem[fx.mem], level[fx.mem]);
        }
    }
}

} // namespace

ExecReport execute(const ModelConfig& model, const HardwareConfig& hw, const SwapPlan& plan,
                   ScheduleVariant variant, const ExecOptions& options,
                   const std::vector<ChunkBuffers>* chunks) {
    ExecReport rep;
    TaskGraph reference = build_schedule(model, hw, plan, variant);
    rep.graph = map_graph_for_b200(reference, options.tier, std::max<std::uint32_t>(2, options.state_slots),
                                   options.resident_groups);
    if (options.swap_only) {
        reference = swap_subgraph(reference, options.max_blocks);
        rep.graph = swap_subgraph(rep.graph, options.max_blocks);
    }
    rep.host_ring = host_ring_depths(rep.graph, options);
    add_host_ring_edges(rep.graph, rep.host_ring);
    for (const Task& t : reference.tasks)
        if (t.kind == TaskKind::transfer)
            rep.reference_bytes[std::string(to_string(t.resource)) + "/" + to_string(t.payload)] += t.work;

    Engine eng(model, plan, rep.graph, options, chunks);
    eng.setup();
    rep.resident_groups = eng.resident_count();
    if (options.resident_groups == kResidentAuto && !options.swap_only) {
        // the engine sized the resident groups from the HBM left free: map
        // again with that count (same tasks and ids; state hops of resident
        // groups now move 0 B and their states are booked up front)
        rep.graph = map_graph_for_b200(reference, options.tier, std::max<std::uint32_t>(2, options.state_slots),
                                       rep.resident_groups);
        add_host_ring_edges(rep.graph, rep.host_ring);
    }
    if (options.tier == StateTier::file) {
        rep.io_engine = eng.io_engine();
        rep.file_devices = static_cast<std::uint32_t>(eng.file_dirs().size());
    }
    rep.file_warmup_s = eng.warm_file_lane();
    MeasuredRates rates = eng.calibrate();
    rep.io_registered_bytes = eng.io_registered();
    const std::uint64_t cal_fixed = eng.io_fixed(), cal_plain = eng.io_plain();
    if (rates.compute_flops <= 0) rates.compute_flops = hw.gpu_tput;
    rep.hw_exec = b200_hardware(hw, rates);
    rep.planned = simulate(rep.graph, rep.hw_exec);
    link_overlap(rep.graph, rep.planned, rates);
    rep.hw_predicted = b200_hardware_effective(hw, rates);
    rep.predicted = simulate(rep.graph, rep.hw_predicted);
    rep.hw_scenario = hw;
    rep.scenario_predicted = simulate(rep.graph, hw);
    rep.rates = rates;
    eng.run(rep.planned, rep);
    rep.io_fixed_requests -= cal_fixed;  // the iteration's requests only
    rep.io_plain_requests -= cal_plain;
    rep.invariants = check_trace_invariants(rep.graph, rep.trace, rep.hw_exec);
    return rep;
}

} // namespace offsim
