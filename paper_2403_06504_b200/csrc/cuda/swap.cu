// Activation swap engine — see swap.cuh.
#include "swap.cuh"

#include "adamw_kernels.cuh"
#include "pipeline.cuh"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <set>

namespace fy {

namespace {

constexpr std::uint64_t kAlign = 4096;  // O_DIRECT granularity
std::uint64_t round_up(std::uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Host function on the IO stream: one file transfer of a ring slot.
void CUDART_CB run_swap_io(void* arg) {
    auto* r = static_cast<Swapper::IoReq*>(arg);
    Swapper& s = *r->self;
    if (s.io_failed.load()) {
        s.io_done.fetch_add(1, std::memory_order_release);
        return;
    }
    std::string err;
    try {
        err = s.engine().transfer(s.stripe(), r->buf, r->bytes, r->offset, r->write);
    } catch (const std::exception& e) {
        err = e.what();
    }
    if (!err.empty()) {
        std::lock_guard<std::mutex> lk(s.io_mu);
        s.io_error = err;
        s.io_failed.store(1);
    }
    s.io_done.fetch_add(1, std::memory_order_release);
}

} // namespace

Swapper::Swapper(const fy_swap_config& cfg) : cfg_(cfg) {
    if (cfg_.slots == 0) cfg_.slots = 4;
    if (cfg_.slot_bytes == 0) cfg_.slot_bytes = 64ull << 20;
    if (cfg_.slots < 2) throw ArgError("swapper: slots must be >= 2");
    cfg_.slot_bytes = round_up(cfg_.slot_bytes);
    // one directory, or several separated by ':' (one per SSD: the swap
    // file is striped RAID-0 over them)
    const std::string dirs = cfg_.file_dir && *cfg_.file_dir ? cfg_.file_dir : "/tmp";
    for (std::size_t a = 0; a <= dirs.size();) {
        const std::size_t b = std::min(dirs.find(':', a), dirs.size());
        if (b > a) dirs_.push_back(dirs.substr(a, b - a));
        a = b + 1;
    }
    if (dirs_.empty() || dirs_.size() > 64) throw ArgError("swapper: file_dir must name 1..64 directories");
    if (std::set<std::string>(dirs_.begin(), dirs_.end()).size() != dirs_.size())
        throw ArgError("swapper: file_dir entries must be distinct");
    try {
        check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
        check_cuda(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "swap d2h stream");
        check_cuda(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "swap h2d stream");
        check_cuda(cudaStreamCreateWithFlags(&io_s_, cudaStreamNonBlocking), "swap io stream");
    } catch (...) {
        release_all();
        throw;
    }
}

Swapper::~Swapper() { release_all(); }

void Swapper::release_all() noexcept {
    cudaSetDevice(cfg_.device);
    if (d2h_) cudaStreamSynchronize(d2h_);
    if (h2d_) cudaStreamSynchronize(h2d_);
    if (io_s_) cudaStreamSynchronize(io_s_);
    (void)io_done.load(std::memory_order_acquire);  // the IO host functions are done
    for (auto& [h, e] : entries_) {
        if (e.stored) cudaEventDestroy(e.stored);
        if (e.host && !host_free(e.host)) cudaFreeHost(e.host);
    }
    entries_.clear();
    for (auto& [cap, p] : free_host_)
        if (!host_free(p)) cudaFreeHost(p);
    free_host_.clear();
    io_.unregister_buffers();
    for (void* p : slots_)
        if (!host_free(p)) cudaFreeHost(p);
    slots_.clear();
    for (cudaEvent_t e : slot_free_) cudaEventDestroy(e);
    for (cudaEvent_t e : slot_filled_) cudaEventDestroy(e);
    slot_free_.clear();
    slot_filled_.clear();
    if (d2h_) cudaStreamDestroy(d2h_);
    if (h2d_) cudaStreamDestroy(h2d_);
    if (io_s_) cudaStreamDestroy(io_s_);
    d2h_ = h2d_ = io_s_ = nullptr;
    close_files();
}

void Swapper::close_files() noexcept {
    for (std::size_t i = 0; i < fds_.size(); ++i) {
        ::close(fds_[i]);
        ::unlink(paths_[i].c_str());
    }
    fds_.clear();
    paths_.clear();
}

void Swapper::open_file() {
    if (!fds_.empty()) return;
    const std::string name = "/fy_swap_" + std::to_string(::getpid()) + "_" +
                             std::to_string(reinterpret_cast<std::uintptr_t>(this)) + ".bin";
    for (const std::string& dir : dirs_) {
        const std::string path = dir + name;
        int flags = O_RDWR | O_CREAT | O_TRUNC;
        if (cfg_.direct_io) flags |= O_DIRECT;
        int fd = ::open(path.c_str(), flags, 0600);
        if (fd < 0 && cfg_.direct_io) fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
        if (fd < 0) {
            const std::string why = std::strerror(errno);
            close_files();
            throw DeviceError("swapper: cannot open " + path + ": " + why);
        }
        fds_.push_back(fd);
        paths_.push_back(path);
    }
    // the pinned ring (SSD placement only); all or nothing
    try {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        for (std::uint32_t i = 0; i < cfg_.slots; ++i) {
            void* p = host_alloc(cfg_.slot_bytes, device_numa_node(dev), nullptr);
            if (!p) check_cuda(cudaHostAlloc(&p, cfg_.slot_bytes, cudaHostAllocPortable), "swap ring");
            slots_.push_back(p);
            cudaEvent_t a, b;
            check_cuda(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
            slot_free_.push_back(a);
            check_cuda(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
            slot_filled_.push_back(b);
        }
        // every file request's host side is a slot: register the ring with
        // io_uring once (READ/WRITE_FIXED; plain ops if the kernel refuses)
        std::vector<std::pair<void*, std::uint64_t>> bufs;
        for (void* p : slots_) bufs.emplace_back(p, cfg_.slot_bytes);
        io_.register_buffers(bufs);
    } catch (...) {
        for (void* p : slots_)
            if (!host_free(p)) cudaFreeHost(p);
        for (cudaEvent_t e : slot_free_) cudaEventDestroy(e);
        for (cudaEvent_t e : slot_filled_) cudaEventDestroy(e);
        slots_.clear();
        slot_free_.clear();
        slot_filled_.clear();
        close_files();
        throw;
    }
}

void* Swapper::take_host(std::uint64_t bytes, std::uint64_t* cap) {
    // reuse a cached pinned buffer of 1x..2x the size, else allocate
    auto it = free_host_.lower_bound(bytes);
    if (it != free_host_.end() && it->first <= 2 * bytes) {
        void* p = it->second;
        *cap = it->first;
        free_host_.erase(it);
        return p;
    }
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    void* p = host_alloc(bytes, device_numa_node(dev), nullptr);
    if (!p) {
        const cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
        if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
        check_cuda(e, "swap host buffer");
    }
    host_bytes_ += bytes;
    *cap = bytes;
    return p;
}

void Swapper::give_host(void* p, std::uint64_t cap) { free_host_.emplace(cap, p); }

std::uint64_t Swapper::swap_out(const void* src, std::uint64_t bytes, int placement, cudaEvent_t ready,
                                cudaEvent_t src_free) {
    if (!src || bytes == 0) throw ArgError("swap_out: null source or zero bytes");
    if (placement != FY_SWAP_CPU && placement != FY_SWAP_SSD) throw ArgError("swap_out: bad placement");
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    if (placement == FY_SWAP_SSD) open_file();  // may throw: before anything is allocated
    Entry e;
    e.bytes = bytes;
    e.placement = placement;
    if (placement == FY_SWAP_CPU) e.host = take_host(bytes, &e.host_cap);  // may throw (host memory)
    if (const cudaError_t err = cudaEventCreateWithFlags(&e.stored, cudaEventDisableTiming); err != cudaSuccess) {
        if (e.host) give_host(e.host, e.host_cap);
        check_cuda(err, "event");
    }
    if (ready) check_cuda(cudaStreamWaitEvent(d2h_, ready, 0), "wait ready");
    if (placement == FY_SWAP_CPU) {
        check_cuda(cudaMemcpyAsync(e.host, src, bytes, cudaMemcpyDeviceToHost, d2h_), "swap out D2H");
        check_cuda(cudaEventRecord(e.stored, d2h_), "record");
    } else {
        e.file_off = file_end_;
        file_end_ += round_up(bytes);
        for (std::uint64_t off = 0; off < bytes; off += cfg_.slot_bytes) {
            const std::uint64_t n = std::min<std::uint64_t>(cfg_.slot_bytes, bytes - off);
            const std::uint32_t s = next_slot_++ % cfg_.slots;
            check_cuda(cudaStreamWaitEvent(d2h_, slot_free_[s], 0), "wait slot");
            check_cuda(cudaMemcpyAsync(slots_[s], static_cast<const char*>(src) + off, n,
                                       cudaMemcpyDeviceToHost, d2h_),
                       "swap out D2H (ring)");
            check_cuda(cudaEventRecord(slot_filled_[s], d2h_), "record");
            check_cuda(cudaStreamWaitEvent(io_s_, slot_filled_[s], 0), "wait filled");
            reqs_.push_back(IoReq{this, slots_[s], round_up(n), e.file_off + off, true});
            check_cuda(cudaLaunchHostFunc(io_s_, run_swap_io, &reqs_.back()), "swap write");
            check_cuda(cudaEventRecord(slot_free_[s], io_s_), "record");
        }
        check_cuda(cudaEventRecord(e.stored, io_s_), "record");
    }
    if (src_free) check_cuda(cudaEventRecord(src_free, d2h_), "record src_free");
    const std::uint64_t h = next_handle_++;
    entries_.emplace(h, e);
    return h;
}

void Swapper::swap_in(std::uint64_t handle, void* dst, cudaEvent_t ready, cudaEvent_t done) {
    const auto it = entries_.find(handle);
    if (it == entries_.end()) throw ArgError("swap_in: unknown handle " + std::to_string(handle));
    if (!dst) throw ArgError("swap_in: null destination");
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    const Entry& e = it->second;
    if (ready) check_cuda(cudaStreamWaitEvent(h2d_, ready, 0), "wait ready");
    if (e.placement == FY_SWAP_CPU) {
        check_cuda(cudaStreamWaitEvent(h2d_, e.stored, 0), "wait stored");
        check_cuda(cudaMemcpyAsync(dst, e.host, e.bytes, cudaMemcpyHostToDevice, h2d_), "swap in H2D");
    } else {
        check_cuda(cudaStreamWaitEvent(io_s_, e.stored, 0), "wait stored");
        for (std::uint64_t off = 0; off < e.bytes; off += cfg_.slot_bytes) {
            const std::uint64_t n = std::min<std::uint64_t>(cfg_.slot_bytes, e.bytes - off);
            const std::uint32_t s = next_slot_++ % cfg_.slots;
            check_cuda(cudaStreamWaitEvent(io_s_, slot_free_[s], 0), "wait slot");
            reqs_.push_back(IoReq{this, slots_[s], round_up(n), e.file_off + off, false});
            check_cuda(cudaLaunchHostFunc(io_s_, run_swap_io, &reqs_.back()), "swap read");
            check_cuda(cudaEventRecord(slot_filled_[s], io_s_), "record");
            check_cuda(cudaStreamWaitEvent(h2d_, slot_filled_[s], 0), "wait filled");
            check_cuda(cudaMemcpyAsync(static_cast<char*>(dst) + off, slots_[s], n, cudaMemcpyHostToDevice,
                                       h2d_),
                       "swap in H2D (ring)");
            check_cuda(cudaEventRecord(slot_free_[s], h2d_), "record");
        }
    }
    if (done) check_cuda(cudaEventRecord(done, h2d_), "record done");
}

void Swapper::release(std::uint64_t handle) {
    const auto it = entries_.find(handle);
    if (it == entries_.end()) throw ArgError("swap_release: unknown handle " + std::to_string(handle));
    Entry e = it->second;
    entries_.erase(it);
    // in-flight copies may still read the buffer: it returns to the cache
    // only after this handle's queued work (a swap_in may follow a release
    // only through a new handle)
    check_cuda(cudaEventSynchronize(e.stored), "release");
    check_cuda(cudaStreamSynchronize(h2d_), "release");
    (void)io_done.load(std::memory_order_acquire);
    cudaEventDestroy(e.stored);
    if (e.host) give_host(e.host, e.host_cap);
    bool any_file = false;
    for (const auto& [h, x] : entries_) any_file = any_file || x.placement == FY_SWAP_SSD;
    if (!any_file) file_end_ = 0;  // every file region is free again
}

void Swapper::sync() {
    check_cuda(cudaSetDevice(cfg_.device), "cudaSetDevice");
    check_cuda(cudaStreamSynchronize(d2h_), "swap sync");
    check_cuda(cudaStreamSynchronize(io_s_), "swap sync");
    check_cuda(cudaStreamSynchronize(h2d_), "swap sync");
    (void)io_done.load(std::memory_order_acquire);  // pairs with run_swap_io's release
    reqs_.clear();
    if (io_failed.load()) {
        std::lock_guard<std::mutex> lk(io_mu);
        const std::string err = io_error;
        io_failed.store(0);
        throw DeviceError("swap file IO: " + err);
    }
}

} // namespace fy
