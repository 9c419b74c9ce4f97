// IoEngine self-test (test infrastructure): writes a patterned buffer to a
// file through the engine (io_uring when available, O_DIRECT), reads it
// back into a second buffer and compares. Prints "<engine> OK <MB/s write>
// <MB/s read>" or an error. Usage: io_engine_test <dir> <MiB> [depth]
#include "../../paper_2403_06504_b200/csrc/core/io_engine.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

// Fault injection (SURVEY.md §5 failure detection): a write through a
// read-only descriptor and a read past the end of a short file must both
// come back as error strings — never a crash, a hang or silent short data.
// Prints "<engine> FAULTS-REPORTED <write error> | <read error>".
static int faults(const std::string& dir, unsigned depth) {
    const std::string path = dir + "/io_engine_fault.bin";
    void* buf = nullptr;
    const std::uint64_t bytes = 8ull << 20;
    if (posix_memalign(&buf, 4096, bytes)) return 3;
    std::memset(buf, 0x5A, bytes);
    int fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
    if (fd < 0) return 4;
    if (::write(fd, buf, 1u << 20) != (1 << 20)) return 5;  // a 1 MiB file
    ::close(fd);
    fy::IoEngine io(depth, 1ull << 20);
    fd = ::open(path.c_str(), O_RDONLY);
    const std::string werr = io.transfer(fd, buf, bytes, 0, true);   // EBADF
    const std::string rerr = io.transfer(fd, buf, bytes, 0, false);  // 7 MiB past EOF
    ::close(fd);
    ::unlink(path.c_str());
    std::free(buf);
    if (werr.empty() || rerr.empty()) {
        std::printf("%s NOT-REPORTED [%s] [%s]\n", io.engine(), werr.c_str(), rerr.c_str());
        return 1;
    }
    std::printf("%s FAULTS-REPORTED %s | %s\n", io.engine(), werr.c_str(), rerr.c_str());
    return 0;
}

// Striping: a logical region at a 12 KiB offset (not unit-aligned) written
// over `count` files with a 1 MiB stripe unit and 256 KiB requests, read back
// through the engine, and every device file checked against the RAID-0
// mapping with plain preads. Prints "<engine> STRIPE-OK <count>".
static int stripe(const std::string& dir, unsigned count, std::uint64_t mib, bool fixed) {
    const std::uint64_t unit = 1ull << 20, bytes = mib << 20, offset = 3 * 4096;
    std::vector<int> fds;
    std::vector<std::string> paths;
    for (unsigned d = 0; d < count; ++d) {
        paths.push_back(dir + "/io_engine_stripe_" + std::to_string(d) + ".bin");
        int fd = ::open(paths.back().c_str(), O_RDWR | O_CREAT | O_TRUNC | O_DIRECT, 0600);
        if (fd < 0) fd = ::open(paths.back().c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
        if (fd < 0) return 4;
        fds.push_back(fd);
    }
    void *a = nullptr, *b = nullptr;
    if (posix_memalign(&a, 4096, bytes) || posix_memalign(&b, 4096, bytes)) return 3;
    auto* pa = static_cast<std::uint64_t*>(a);
    for (std::uint64_t i = 0; i < bytes / 8; ++i) pa[i] = (i + 17) * 0x9e3779b97f4a7c15ull;
    std::memset(b, 0, bytes);
    fy::IoEngine io(8, 256ull << 10);
    if (fixed) io.register_buffers({{a, bytes}, {b, bytes}});
    const fy::IoEngine::Stripe st{fds.data(), count, unit};
    std::string err = io.transfer(st, a, bytes, offset, true);
    if (err.empty()) err = io.transfer(st, b, bytes, offset, false);
    bool ok = err.empty() && std::memcmp(a, b, bytes) == 0;
    // the layout itself: logical byte o -> file (o / unit) % count
    for (unsigned d = 0; d < count; ++d) ::close(fds[d]);
    std::vector<char> page(4096);
    for (std::uint64_t o = offset; ok && o < offset + bytes; o += 4096) {
        const std::uint64_t s = o / unit;
        const int fd = ::open(paths[s % count].c_str(), O_RDONLY);
        const off_t dev_off = static_cast<off_t>((s / count) * unit + o % unit);
        ok = fd >= 0 && ::pread(fd, page.data(), 4096, dev_off) == 4096 &&
             std::memcmp(page.data(), static_cast<char*>(a) + (o - offset), 4096) == 0;
        if (fd >= 0) ::close(fd);
    }
    for (const auto& p : paths) ::unlink(p.c_str());
    std::free(a);
    std::free(b);
    if (!ok) {
        std::printf("%s STRIPE-MISMATCH %s\n", io.engine(), err.c_str());
        return 1;
    }
    std::printf("%s STRIPE-OK %u fixed=%llu plain=%llu\n", io.engine(), count,
                static_cast<unsigned long long>(io.fixed_requests()),
                static_cast<unsigned long long>(io.plain_requests()));
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    if (std::string(argv[2]) == "fault") return faults(argv[1], argc > 3 ? std::atoi(argv[3]) : 8);
    if (std::string(argv[2]) == "stripe")
        return stripe(argv[1], argc > 3 ? std::atoi(argv[3]) : 3, argc > 4 ? std::atoi(argv[4]) : 7,
                      argc > 5 && std::string(argv[5]) == "fixed");
    const std::string path = std::string(argv[1]) + "/io_engine_test.bin";
    const std::uint64_t bytes = std::strtoull(argv[2], nullptr, 10) << 20;
    const unsigned depth = argc > 3 ? static_cast<unsigned>(std::atoi(argv[3])) : 32;
    void *a = nullptr, *b = nullptr;
    if (posix_memalign(&a, 4096, bytes) || posix_memalign(&b, 4096, bytes)) return 3;
    auto* pa = static_cast<std::uint64_t*>(a);
    for (std::uint64_t i = 0; i < bytes / 8; ++i) pa[i] = i * 0x9e3779b97f4a7c15ull;
    std::memset(b, 0, bytes);
    int fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC | O_DIRECT, 0600);
    if (fd < 0) fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
    if (fd < 0) return 4;
    fy::IoEngine io(depth, 1ull << 20);
    // "fixed": register both buffers (b in two halves) -> READ/WRITE_FIXED
    const bool fixed = argc > 4 && std::string(argv[4]) == "fixed";
    std::uint64_t reg = 0;
    if (fixed)
        reg = io.register_buffers({{a, bytes}, {b, bytes / 2}, {static_cast<char*>(b) + bytes / 2, bytes - bytes / 2}});
    const auto t0 = std::chrono::steady_clock::now();
    std::string err = io.transfer(fd, a, bytes, 0, true);
    const auto t1 = std::chrono::steady_clock::now();
    if (err.empty()) err = io.transfer(fd, b, bytes, 0, false);
    const auto t2 = std::chrono::steady_clock::now();
    ::close(fd);
    ::unlink(path.c_str());
    if (!err.empty()) {
        std::printf("%s ERROR %s\n", io.engine(), err.c_str());
        return 1;
    }
    const bool same = std::memcmp(a, b, bytes) == 0;
    const double w = bytes / 1e6 / std::chrono::duration<double>(t1 - t0).count();
    const double r = bytes / 1e6 / std::chrono::duration<double>(t2 - t1).count();
    std::printf("%s %s %.0f %.0f fixed=%llu plain=%llu registered=%llu\n", io.engine(), same ? "OK" : "MISMATCH", w,
                r, static_cast<unsigned long long>(io.fixed_requests()),
                static_cast<unsigned long long>(io.plain_requests()), static_cast<unsigned long long>(reg));
    return same ? 0 : 1;
}
