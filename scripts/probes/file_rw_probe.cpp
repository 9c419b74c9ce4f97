// Probe (r02aq): why do the C5 swap sweep's file READ legs run at 0.55-0.69
// of the run's own replayed read rate on the lease's virtio disk?
// Mimics the swap-only iteration's file lane with the product's IoEngine
// (O_DIRECT io_uring, 32 x 4 MiB in flight): write `blocks` checkpoints of
// `size` bytes in forward order, then read them back in reverse (backward)
// order — (a) right after the writes, (b) after an fsync + pause, (c) again
// (a second read of the same data). argv: dir blocks size pause_s random(0/1)
// — random = incompressible buffer contents instead of a constant fill. Prints one JSON line per phase:
// GB/s over the phase and min / median / max per request.
// Build: g++ -O2 -std=c++20 -Ipaper_2403_06504_b200/csrc/core -I/usr/local/cuda/include \
//        scripts/probes/file_rw_probe.cpp paper_2403_06504_b200/csrc/core/io_engine.cpp \
//        -L/usr/local/cuda/lib64 -lcudart
// argv[6] distinct (0/1), argv[7] pinned (0/1), argv[8] link_load (0/1).
#include "io_engine.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {
double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void report(const char* phase, const std::vector<double>& t, std::uint64_t size) {
    std::vector<double> s = t;
    std::sort(s.begin(), s.end());
    double total = 0;
    for (double x : t) total += x;
    std::printf("{\"phase\": \"%s\", \"requests\": %zu, \"gbs\": %.3f, \"req_ms_min\": %.2f, "
                "\"req_ms_med\": %.2f, \"req_ms_max\": %.2f}\n",
                phase, t.size(), size * t.size() / total / 1e9, s.front() * 1e3, s[s.size() / 2] * 1e3,
                s.back() * 1e3);
    std::fflush(stdout);
}
} // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    const int blocks = argc > 2 ? std::atoi(argv[2]) : 40;
    const std::uint64_t size = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 83886080ull;
    const int pause_s = argc > 4 ? std::atoi(argv[4]) : 20;
    const bool random_data = argc > 5 && std::atoi(argv[5]) != 0;
    // distinct: every block has its own buffer region (like the executor's
    // per-checkpoint host copies) instead of one reused buffer; pinned: the
    // buffer is a MADV_HUGEPAGE mmap registered with cudaHostRegister (like
    // fy::host_alloc)
    const bool distinct = argc > 6 && std::atoi(argv[6]) != 0;
    const bool pinned = argc > 7 && std::atoi(argv[7]) != 0;
    // link_load: a second thread keeps the GPU copy engines busy the whole
    // time (1 = H2D + D2H 256 MiB copies from / to pinned host memory,
    // back to back), as the executed iteration's copies are beside its file IO
    const int link_load = argc > 8 ? std::atoi(argv[8]) : 0;
    const std::string path = dir + "/file_rw_probe.bin";
    int fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC | O_DIRECT, 0600);
    if (fd < 0) {
        std::perror("open");
        return 1;
    }
    const std::uint64_t total = distinct ? size * blocks : size;
    void* buf = nullptr;
    if (pinned) {
        buf = ::mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (buf == MAP_FAILED) return 1;
        ::madvise(buf, total, MADV_HUGEPAGE);
    } else if (posix_memalign(&buf, 4096, total)) {
        return 1;
    }
    std::memset(buf, 0x5A, total);
    if (pinned && cudaHostRegister(buf, total, cudaHostRegisterPortable) != cudaSuccess) return 3;
    if (random_data) {  // incompressible contents (xorshift64), like real activations
        std::uint64_t x = 0x9E3779B97F4A7C15ull;
        auto* q = static_cast<std::uint64_t*>(buf);
        for (std::uint64_t i = 0; i < total / 8; ++i) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            q[i] = x;
        }
    }
    std::atomic<bool> stop{false};
    std::atomic<std::uint64_t> link_bytes{0};
    std::thread loader;
    if (link_load) {
        loader = std::thread([&] {
            const std::size_t lb = 256ull << 20;
            void *hu = nullptr, *hd = nullptr, *du = nullptr, *dd = nullptr;
            cudaHostAlloc(&hu, lb, cudaHostAllocDefault);
            cudaHostAlloc(&hd, lb, cudaHostAllocDefault);
            cudaMalloc(&du, lb);
            cudaMalloc(&dd, lb);
            cudaStream_t su, sd;
            cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
            while (!stop.load()) {
                cudaMemcpyAsync(du, hu, lb, cudaMemcpyHostToDevice, su);
                cudaMemcpyAsync(hd, dd, lb, cudaMemcpyDeviceToHost, sd);
                cudaStreamSynchronize(su);
                cudaStreamSynchronize(sd);
                link_bytes += 2 * lb;
            }
            cudaFree(du);
            cudaFree(dd);
            cudaFreeHost(hu);
            cudaFreeHost(hd);
        });
        std::this_thread::sleep_for(std::chrono::milliseconds(200));
    }
    const double l0 = now();
    fy::IoEngine io(32, 4ull << 20);
    std::printf("{\"engine\": \"%s\", \"blocks\": %d, \"size\": %llu, \"random_data\": %d, \"distinct\": %d, "
                "\"pinned\": %d, \"link_load\": %d}\n", io.engine(), blocks, static_cast<unsigned long long>(size), random_data ? 1 : 0,
                distinct ? 1 : 0, pinned ? 1 : 0, link_load);
    auto run = [&](const char* phase, bool write, bool reverse) {
        std::vector<double> t;
        for (int i = 0; i < blocks; ++i) {
            const int k = reverse ? blocks - 1 - i : i;
            const double t0 = now();
            char* b = static_cast<char*>(buf) + (distinct ? static_cast<std::uint64_t>(k) * size : 0);
            const std::string err = io.transfer(fd, b, size, static_cast<std::uint64_t>(k) * size, write);
            t.push_back(now() - t0);
            if (!err.empty()) {
                std::fprintf(stderr, "%s\n", err.c_str());
                std::exit(2);
            }
        }
        report(phase, t, size);
    };
    run("write_1", true, false);
    run("read_right_after_write", false, true);
    run("write_2", true, false);
    const double f0 = now();
    ::fsync(fd);
    std::printf("{\"phase\": \"fsync\", \"s\": %.3f}\n", now() - f0);
    std::this_thread::sleep_for(std::chrono::seconds(pause_s));
    run("read_after_fsync_pause", false, true);
    run("read_again", false, true);
    run("read_forward_order", false, false);
    if (link_load) {
        stop = true;
        loader.join();
        std::printf("{\"link_load_gbs_both_ways\": %.2f}\n", link_bytes.load() / (now() - l0) / 1e9);
    }
    ::close(fd);
    ::unlink(path.c_str());
    if (pinned) {
        cudaHostUnregister(buf);
        ::munmap(buf, total);
    } else {
        std::free(buf);
    }
    return 0;
}
