// File-tier IO engine: io_uring on raw syscalls (liburing is not available):
// submits one large transfer as many fixed-size O_DIRECT reads/writes in
// flight at once, which is what an NVMe array needs to reach its aggregate
// bandwidth (the reference's SSD lane is n_ssd devices, hardware.cpp:39-42).
// Falls back to a pread/pwrite loop when io_uring_setup is refused (old
// kernel or a sandbox seccomp policy); `engine()` reports which one ran.
// Long-lived staging buffers (the executor's pinned rings, the swap
// engine's slots) can be registered with the ring once: requests that fall
// inside them go out as READ_FIXED / WRITE_FIXED, so the kernel does not
// pin and unpin the pages of every request.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace fy {

class IoEngine {
public:
    // depth: requests in flight; piece: bytes per request (multiple of 4 KiB)
    explicit IoEngine(unsigned depth = 32, std::uint64_t piece = 4ull << 20);
    ~IoEngine();
    IoEngine(const IoEngine&) = delete;
    IoEngine& operator=(const IoEngine&) = delete;

    // Transfers `bytes` between buf and fd at `offset`; returns "" on
    // success or an error message. Thread-compatible (one caller at a time).
    std::string transfer(int fd, void* buf, std::uint64_t bytes, std::uint64_t offset, bool write);

    // A logical file striped over `count` files (one per device): logical
    // byte o lives in fds[(o / unit) % count] at ((o / unit) / count) * unit
    // + o % unit — RAID-0 over the reference's n_ssd devices
    // (hardware.cpp:39-42 aggregates their bandwidth). One ring drives all
    // of them, so every device has requests in flight at once.
    struct Stripe {
        const int* fds;
        unsigned count;
        std::uint64_t unit; // multiple of 4 KiB
    };
    std::string transfer(const Stripe& st, void* buf, std::uint64_t bytes, std::uint64_t offset, bool write);

    const char* engine() const { return ring_fd_ >= 0 ? "io_uring" : "pread/pwrite"; }

    // Registers (base, bytes) buffers, replacing any earlier registration;
    // each is split into <= 1 GiB pieces (the kernel's per-buffer limit).
    // Returns the registered bytes (0 on the fallback engine or when the
    // kernel refuses, e.g. RLIMIT_MEMLOCK; transfers then use plain ops).
    std::uint64_t register_buffers(const std::vector<std::pair<void*, std::uint64_t>>& bufs);
    void unregister_buffers();
    // requests issued so far as fixed-buffer / plain io_uring ops
    std::uint64_t fixed_requests() const { return fixed_requests_; }
    std::uint64_t plain_requests() const { return plain_requests_; }

private:
    std::string transfer_sync(int fd, void* buf, std::uint64_t bytes, std::uint64_t offset, bool write);
    struct Req {
        int fd;
        char* buf;
        std::uint64_t len, off;
    };
    std::string submit(const std::vector<Req>& reqs, bool write);

    int ring_fd_ = -1;
    unsigned depth_ = 0;
    std::uint64_t piece_ = 0;
    // mapped rings
    void* sq_ptr_ = nullptr;
    void* cq_ptr_ = nullptr;
    void* sqes_ = nullptr;
    std::uint64_t sq_len_ = 0, cq_len_ = 0, sqes_len_ = 0;
    unsigned* sq_head_ = nullptr;
    unsigned* sq_tail_ = nullptr;
    unsigned* sq_mask_ = nullptr;
    unsigned* sq_array_ = nullptr;
    unsigned* cq_head_ = nullptr;
    unsigned* cq_tail_ = nullptr;
    unsigned* cq_mask_ = nullptr;
    void* cqes_ = nullptr;
    struct Region {
        std::uint64_t base, len;
        unsigned index;
    };
    std::vector<Region> regions_; // sorted by base
    std::uint64_t fixed_requests_ = 0, plain_requests_ = 0;
    // index of the registered buffer holding [p, p + len), or -1
    int fixed_index(std::uint64_t p, std::uint64_t len) const;
};

} // namespace fy
