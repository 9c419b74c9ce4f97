// NUMA-local pinned host memory for the optimizer's host tier.
//
// The north star shards the step across the GPUs of one box with "each GPU
// updating its own shard from NUMA-local pinned memory": on a two-socket
// 8xB200 server, states pinned on the far socket cross the inter-socket link
// on every H2D/D2H. cudaHostAlloc places pages wherever the calling thread
// first touches them, so instead the allocation is an anonymous mapping with
// a MPOL_PREFERRED policy for the GPU's NUMA node (read from the PCI sysfs
// node of the device), populated under that policy, then page-locked with
// cudaHostRegister (portable). Raw syscalls: no libnuma dependency. On a
// one-node host (or when sysfs reports -1) this degrades to an ordinary
// registered allocation.
#include "adamw_kernels.cuh"

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace fy {

namespace {

constexpr int kMpolPreferred = 1;
constexpr std::uint64_t kHuge = 2ull << 20;

struct Mapping {
    std::uint64_t len;
    bool registered;
};
std::mutex g_mu;
std::map<void*, Mapping> g_maps;

std::uint64_t round_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

// Populate the pages from several threads (first touch under the policy);
// for tens of GB a single-threaded fault-in dominates allocation time.
void populate(unsigned char* p, std::uint64_t len) {
    const long page = ::sysconf(_SC_PAGESIZE);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nt = len >= (1ull << 30) ? hw : 1;
    std::vector<std::thread> th;
    const std::uint64_t per = round_up((len + nt - 1) / nt, static_cast<std::uint64_t>(page));
    for (unsigned t = 0; t < nt; ++t) {
        const std::uint64_t lo = t * per, hi = std::min(len, lo + per);
        if (lo >= hi) break;
        th.emplace_back([=] {
            for (std::uint64_t o = lo; o < hi; o += static_cast<std::uint64_t>(page)) p[o] = 0;
        });
    }
    for (auto& t : th) t.join();
}

} // namespace

int device_numa_node(int device) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string id(bus);
    for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    // sysfs uses a 4-hex-digit domain ("0000:1b:00.0"); the runtime may
    // report 8 ("00000000:1B:00.0")
    if (id.size() > 12 && id.find(':') == 8) id = id.substr(4);
    std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
    int node = -1;
    if (!(f >> node)) return -1;
    return node;
}

int host_numa_node(const void* p) {
    void* page = const_cast<void*>(p);
    int status = -1;
    if (::syscall(SYS_move_pages, 0, 1UL, &page, nullptr, &status, 0) != 0) return -1;
    return status;  // node, or -errno for an unpopulated page
}

std::uint64_t host_mem_available() {
    std::ifstream f("/proc/meminfo");
    std::string key;
    std::uint64_t kb = 0;
    std::string unit;
    while (f >> key >> kb) {
        std::getline(f, unit);
        if (key == "MemAvailable:") return kb * 1024ull;
    }
    return ~0ull;  // unknown: let mmap / cudaHostRegister decide
}

void* host_alloc(std::uint64_t bytes, int node, int* placed) {
    const std::uint64_t len = round_up(std::max<std::uint64_t>(bytes, 1), kHuge);
    // populate() touches every page, so an oversized request would be
    // OOM-killed instead of failing: refuse it here (nullptr -> the caller's
    // FY_ERR_INFEASIBLE / cudaHostAlloc fallback), keeping 1 GiB of headroom.
    const std::uint64_t avail = host_mem_available();
    if (avail != ~0ull && len + (1ull << 30) > avail) return nullptr;
    void* p = ::mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    ::madvise(p, len, MADV_HUGEPAGE);  // fewer pages to pin (best effort)
    bool bound = false;
    if (node >= 0 && node < 1024) {
        unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
        mask[node / (8 * sizeof(unsigned long))] |= 1UL << (node % (8 * sizeof(unsigned long)));
        bound = ::syscall(SYS_mbind, p, len, kMpolPreferred, mask, 1024UL, 0U) == 0;
    }
    populate(static_cast<unsigned char*>(p), len);
    const cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ::munmap(p, len);
        return nullptr;
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_maps[p] = Mapping{len, true};
    }
    if (placed) *placed = bound ? host_numa_node(p) : -1;
    return p;
}

bool host_free(void* p) {
    Mapping m{};
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const auto it = g_maps.find(p);
        if (it == g_maps.end()) return false;
        m = it->second;
        g_maps.erase(it);
    }
    if (m.registered) cudaHostUnregister(p);
    ::munmap(p, m.len);
    return true;
}

} // namespace fy
