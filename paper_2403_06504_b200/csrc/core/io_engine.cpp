// io_uring IO engine (raw syscalls) with a pread/pwrite fallback.
#include "io_engine.hpp"

#include <linux/io_uring.h>
#include <sys/mman.h>
#include <sys/uio.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <vector>

namespace fy {

namespace {

int uring_setup(unsigned entries, io_uring_params* p) {
    return static_cast<int>(::syscall(__NR_io_uring_setup, entries, p));
}
int uring_enter(int fd, unsigned submit, unsigned wait, unsigned flags) {
    return static_cast<int>(::syscall(__NR_io_uring_enter, fd, submit, wait, flags, nullptr, 0));
}
int uring_register(int fd, unsigned op, const void* arg, unsigned n) {
    return static_cast<int>(::syscall(__NR_io_uring_register, fd, op, arg, n));
}
template <typename T>
T* at(void* base, std::uint32_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

} // namespace

IoEngine::IoEngine(unsigned depth, std::uint64_t piece)
    // IORING_MAX_ENTRIES is 32768: io_depth x tier devices may exceed it
    : depth_(std::min(std::max(depth, 1u), 32768u)), piece_(piece) {
    io_uring_params p;
    std::memset(&p, 0, sizeof p);
    p.flags = IORING_SETUP_CLAMP;
    const int fd = uring_setup(depth_, &p);
    if (fd < 0) return; // refused: fall back to pread/pwrite
    sq_len_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
    cq_len_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
    const bool single = (p.features & IORING_FEAT_SINGLE_MMAP) != 0;
    if (single) sq_len_ = cq_len_ = std::max(sq_len_, cq_len_);
    sq_ptr_ = ::mmap(nullptr, sq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd,
                     IORING_OFF_SQ_RING);
    if (sq_ptr_ == MAP_FAILED) {
        ::close(fd);
        sq_ptr_ = nullptr;
        return;
    }
    cq_ptr_ = single ? sq_ptr_
                     : ::mmap(nullptr, cq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd,
                              IORING_OFF_CQ_RING);
    sqes_len_ = p.sq_entries * sizeof(io_uring_sqe);
    sqes_ = ::mmap(nullptr, sqes_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd,
                   IORING_OFF_SQES);
    if (cq_ptr_ == MAP_FAILED || sqes_ == MAP_FAILED) {
        ::close(fd);
        return;
    }
    sq_head_ = at<unsigned>(sq_ptr_, p.sq_off.head);
    sq_tail_ = at<unsigned>(sq_ptr_, p.sq_off.tail);
    sq_mask_ = at<unsigned>(sq_ptr_, p.sq_off.ring_mask);
    sq_array_ = at<unsigned>(sq_ptr_, p.sq_off.array);
    cq_head_ = at<unsigned>(cq_ptr_, p.cq_off.head);
    cq_tail_ = at<unsigned>(cq_ptr_, p.cq_off.tail);
    cq_mask_ = at<unsigned>(cq_ptr_, p.cq_off.ring_mask);
    cqes_ = at<void>(cq_ptr_, p.cq_off.cqes);
    depth_ = std::min(depth_, p.sq_entries);
    ring_fd_ = fd;
}

IoEngine::~IoEngine() {
    unregister_buffers();
    if (sqes_ && sqes_ != MAP_FAILED) ::munmap(sqes_, sqes_len_);
    if (cq_ptr_ && cq_ptr_ != MAP_FAILED && cq_ptr_ != sq_ptr_) ::munmap(cq_ptr_, cq_len_);
    if (sq_ptr_ && sq_ptr_ != MAP_FAILED) ::munmap(sq_ptr_, sq_len_);
    if (ring_fd_ >= 0) ::close(ring_fd_);
}

std::uint64_t IoEngine::register_buffers(const std::vector<std::pair<void*, std::uint64_t>>& bufs) {
    unregister_buffers();
    if (ring_fd_ < 0) return 0;
    constexpr std::uint64_t kMaxPiece = 1ull << 30;
    std::vector<iovec> iov;
    std::vector<Region> regions;
    for (const auto& [p, bytes] : bufs) {
        for (std::uint64_t off = 0; off < bytes; off += kMaxPiece) {
            const std::uint64_t len = std::min(kMaxPiece, bytes - off);
            iov.push_back(iovec{static_cast<char*>(p) + off, static_cast<std::size_t>(len)});
            regions.push_back(Region{reinterpret_cast<std::uint64_t>(p) + off, len,
                                     static_cast<unsigned>(iov.size() - 1)});
        }
    }
    if (iov.empty()) return 0;
    if (uring_register(ring_fd_, IORING_REGISTER_BUFFERS, iov.data(), static_cast<unsigned>(iov.size())) < 0)
        return 0;
    std::sort(regions.begin(), regions.end(), [](const Region& a, const Region& b) { return a.base < b.base; });
    regions_ = std::move(regions);
    std::uint64_t total = 0;
    for (const Region& r : regions_) total += r.len;
    return total;
}

void IoEngine::unregister_buffers() {
    if (ring_fd_ >= 0 && !regions_.empty()) uring_register(ring_fd_, IORING_UNREGISTER_BUFFERS, nullptr, 0);
    regions_.clear();
}

int IoEngine::fixed_index(std::uint64_t p, std::uint64_t len) const {
    auto it = std::upper_bound(regions_.begin(), regions_.end(), p,
                               [](std::uint64_t x, const Region& r) { return x < r.base; });
    if (it == regions_.begin()) return -1;
    --it;
    return p + len <= it->base + it->len ? static_cast<int>(it->index) : -1;
}

std::string IoEngine::transfer_sync(int fd, void* buf, std::uint64_t bytes, std::uint64_t offset,
                                    bool write) {
    std::uint64_t done = 0;
    while (done < bytes) {
        char* p = static_cast<char*>(buf) + done;
        const ssize_t n = write ? ::pwrite(fd, p, bytes - done, static_cast<off_t>(offset + done))
                                : ::pread(fd, p, bytes - done, static_cast<off_t>(offset + done));
        if (n < 0 && errno == EINTR) continue;
        if (n <= 0)
            return std::string(write ? "pwrite" : "pread") + " failed: " +
                   (n < 0 ? std::strerror(errno) : "short transfer");
        done += static_cast<std::uint64_t>(n);
    }
    return {};
}

std::string IoEngine::transfer(int fd, void* buf, std::uint64_t bytes, std::uint64_t offset,
                               bool write) {
    const Stripe one{&fd, 1, ~0ull};
    return transfer(one, buf, bytes, offset, write);
}

std::string IoEngine::transfer(const Stripe& st, void* buf, std::uint64_t bytes, std::uint64_t offset,
                               bool write) {
    // split at stripe-unit boundaries (device changes) and at piece_ (the
    // request size), then keep up to depth_ requests in flight
    std::vector<Req> reqs;
    char* p = static_cast<char*>(buf);
    for (std::uint64_t o = offset, end = offset + bytes; o < end;) {
        int fd = st.fds[0];
        std::uint64_t dev_off = o, seg = end - o;
        if (st.count > 1) {
            const std::uint64_t s = o / st.unit, in = o % st.unit;
            fd = st.fds[s % st.count];
            dev_off = (s / st.count) * st.unit + in;
            seg = std::min(seg, st.unit - in);
        }
        for (std::uint64_t done = 0; done < seg;) {
            const std::uint64_t len = std::min(piece_, seg - done);
            reqs.push_back(Req{fd, p + (o - offset) + done, len, dev_off + done});
            done += len;
        }
        o += seg;
    }
    if (ring_fd_ < 0) {
        for (const Req& r : reqs) {
            const std::string err = transfer_sync(r.fd, r.buf, r.len, r.off, write);
            if (!err.empty()) return err;
        }
        return {};
    }
    return submit(reqs, write);
}

std::string IoEngine::submit(const std::vector<Req>& reqs, bool write) {
    const std::uint64_t pieces = reqs.size();
    auto* sqes = static_cast<io_uring_sqe*>(sqes_);
    auto* cqes = static_cast<io_uring_cqe*>(cqes_);
    std::vector<std::uint64_t> short_pieces;
    std::uint64_t next = 0, inflight = 0, failed_errno = 0;
    unsigned unsubmitted = 0; // SQEs past the tail the kernel has not consumed yet
    while (next < pieces || inflight > 0 || unsubmitted > 0) {
        unsigned queued = 0;
        unsigned tail = __atomic_load_n(sq_tail_, __ATOMIC_RELAXED);
        while (next < pieces && inflight + unsubmitted + queued < depth_) {
            const Req& q = reqs[next];
            const unsigned idx = tail & *sq_mask_;
            io_uring_sqe& e = sqes[idx];
            std::memset(&e, 0, sizeof e);
            e.fd = q.fd;
            e.addr = reinterpret_cast<std::uint64_t>(q.buf);
            e.len = static_cast<std::uint32_t>(q.len);
            e.off = q.off;
            const int fixed = regions_.empty() ? -1 : fixed_index(e.addr, e.len);
            if (fixed >= 0) {
                e.opcode = write ? IORING_OP_WRITE_FIXED : IORING_OP_READ_FIXED;
                e.buf_index = static_cast<std::uint16_t>(fixed);
                ++fixed_requests_;
            } else {
                e.opcode = write ? IORING_OP_WRITE : IORING_OP_READ;
                ++plain_requests_;
            }
            e.user_data = next;
            sq_array_[idx] = idx;
            ++tail;
            ++queued;
            ++next;
        }
        __atomic_store_n(sq_tail_, tail, __ATOMIC_RELEASE);
        unsubmitted += queued;
        // consumed SQEs become in flight; a partial submit (or EINTR) leaves
        // the rest in the ring for the next enter
        const int r = uring_enter(ring_fd_, unsubmitted, inflight + unsubmitted > 0 ? 1 : 0,
                                  IORING_ENTER_GETEVENTS);
        if (r < 0 && errno != EINTR && errno != EAGAIN && errno != EBUSY)
            return std::string("io_uring_enter failed: ") + std::strerror(errno);
        const unsigned consumed = r > 0 ? std::min<unsigned>(static_cast<unsigned>(r), unsubmitted) : 0;
        unsubmitted -= consumed;
        inflight += consumed;
        unsigned head = __atomic_load_n(cq_head_, __ATOMIC_RELAXED);
        const unsigned ctail = __atomic_load_n(cq_tail_, __ATOMIC_ACQUIRE);
        while (head != ctail) {
            const io_uring_cqe& c = cqes[head & *cq_mask_];
            const std::uint64_t i = c.user_data;
            if (c.res < 0) failed_errno = static_cast<std::uint64_t>(-c.res);
            else if (static_cast<std::uint64_t>(c.res) != reqs[i].len) short_pieces.push_back(i);
            ++head;
            --inflight;
        }
        __atomic_store_n(cq_head_, head, __ATOMIC_RELEASE);
    }
    if (failed_errno)
        return std::string(write ? "io_uring write" : "io_uring read") + " failed: " +
               std::strerror(static_cast<int>(failed_errno));
    for (const std::uint64_t i : short_pieces) { // rare: finish synchronously
        const Req& q = reqs[i];
        const std::string err = transfer_sync(q.fd, q.buf, q.len, q.off, write);
        if (!err.empty()) return err;
    }
    return {};
}

} // namespace fy
