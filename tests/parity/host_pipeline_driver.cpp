// Native driver of the GPU host-side machinery through the C ABIs only —
// built with -fsanitize=thread by scripts/tsan_gpu.sh (TSAN on
// the host pipeline) and run on a B200 box. Exercises the code paths that
// involve more than one host thread: CUDA host-function callbacks doing
// file IO (executor file tier, swap engine SSD placement), the io_uring
// engine, the chunk pipeline's event chains and the thread-local last error
// used from several threads at once. Exit code 0 = every check passed.
#include "fuyou/fy_adam.h"
#include "offsim/offsim_c.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#define CHECK(x)                                                                     \
    do {                                                                             \
        if (!(x)) {                                                                  \
            std::fprintf(stderr, "FAIL %s:%d %s (%s)\n", __FILE__, __LINE__, #x,     \
                         fy_last_error());                                           \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static int pipeline_case() {
    const uint64_t n = (1u << 22) + 8;
    const int chunks = 6;
    std::vector<void*> hs(chunks), hp(chunks);
    std::vector<void*> dg(chunks);
    for (int k = 0; k < chunks; ++k) {
        CHECK(fy_host_alloc(12 * n, &hs[k]) == FY_OK);
        CHECK(fy_host_alloc(2 * n, &hp[k]) == FY_OK);
        std::memset(hs[k], 0, 12 * n);
        CHECK(cudaMalloc(&dg[k], 2 * n) == cudaSuccess);
        CHECK(cudaMemset(dg[k], 0x3A, 2 * n) == cudaSuccess);
    }
    fy_pipeline_config cfg{};
    cfg.device = 0;
    cfg.max_chunk_elems = n;
    cfg.slots = 3;
    cfg.grad_dtype = FY_BF16;
    cfg.param_dtype = FY_BF16;
    cfg.params_to_host = 1;
    fy_pipeline* p = nullptr;
    CHECK(fy_pipeline_create(&cfg, &p) == FY_OK);
    std::vector<fy_chunk> cs(chunks);
    for (int k = 0; k < chunks; ++k) {
        std::memset(&cs[k], 0, sizeof(fy_chunk));
        cs[k].n = n;
        cs[k].h_states = hs[k];
        cs[k].grad = dg[k];
        cs[k].h_param = hp[k];
    }
    fy_adam_hparams hpar{1e-4f, 0.9f, 0.95f, 1e-8f, 0.1f, 10, 1, 1, 1.0f};
    for (int step = 0; step < 3; ++step) {
        hpar.step = 10 + step;
        CHECK(fy_pipeline_step(p, cs.data(), chunks, &hpar, 1) == FY_OK);
        double sq = 0;
        int bad = 0;
        CHECK(fy_pipeline_wait(p, &sq, &bad) == FY_OK);
        CHECK(sq > 0 && bad == 0);
    }
    fy_pipeline_destroy(p);
    for (int k = 0; k < chunks; ++k) {
        fy_host_free(hs[k]);
        fy_host_free(hp[k]);
        cudaFree(dg[k]);
    }
    return 0;
}

static int swap_case(const char* dir) {
    fy_swap_config sc{0, 1u << 20, 3, dir, 1};
    fy_swapper* s = nullptr;
    CHECK(fy_swapper_create(&sc, &s) == FY_OK);
    const uint64_t sizes[] = {4096, 3 * (1u << 20) + 17, 5u << 20};
    std::vector<void*> src, dst;
    std::vector<uint64_t> h;
    for (int placement = 0; placement < 2; ++placement) {
        for (uint64_t b : sizes) {
            void *a = nullptr, *d = nullptr;
            CHECK(cudaMalloc(&a, b) == cudaSuccess && cudaMalloc(&d, b) == cudaSuccess);
            CHECK(cudaMemset(a, static_cast<int>(b & 0xFF), b) == cudaSuccess);
            CHECK(cudaMemset(d, 0, b) == cudaSuccess);
            src.push_back(a);
            dst.push_back(d);
        }
        CHECK(cudaDeviceSynchronize() == cudaSuccess);
        for (size_t i = 0; i < 3; ++i) {
            uint64_t hh = 0;
            CHECK(fy_swap_out(s, src[src.size() - 3 + i], sizes[i], placement, nullptr, nullptr, &hh) == FY_OK);
            h.push_back(hh);
        }
        for (size_t i = 0; i < 3; ++i)
            CHECK(fy_swap_in(s, h[h.size() - 3 + i], dst[dst.size() - 3 + i], nullptr, nullptr) == FY_OK);
        CHECK(fy_swapper_sync(s) == FY_OK);
    }
    for (size_t i = 0; i < src.size(); ++i) {
        const uint64_t b = sizes[i % 3];
        std::vector<unsigned char> x(b), y(b);
        CHECK(cudaMemcpy(x.data(), src[i], b, cudaMemcpyDeviceToHost) == cudaSuccess);
        CHECK(cudaMemcpy(y.data(), dst[i], b, cudaMemcpyDeviceToHost) == cudaSuccess);
        CHECK(x == y);
        cudaFree(src[i]);
        cudaFree(dst[i]);
    }
    for (uint64_t hh : h) CHECK(fy_swap_release(s, hh) == FY_OK);
    fy_swapper_destroy(s);
    return 0;
}

static int executor_case(const char* dir) {
    const char* sc =
        "{\"schema_version\": 1, \"model\": {\"name\": \"tsan\", \"num_layers\": 4, \"num_heads\": 12, "
        "\"hidden_dim\": 768, \"batch_size\": 8, \"seq_len\": 1024}, \"hardware\": \"a100-12ssd\", "
        "\"variant\": \"overlapped\"}";
    offsim_scenario* s = nullptr;
    CHECK(offsim_scenario_parse(sc, &s) == OFFSIM_OK);
    const std::string opts = std::string("{\"tier\": \"file\", \"host_ring\": 2, \"placement\": \"ssd\", "
                                         "\"file_dir\": \"") + dir + "\"}";
    char* summary = nullptr;
    const offsim_status st = offsim_execute(s, opts.c_str(), &summary, nullptr);
    const auto pass = [](const char* j) {
        return j && (std::strstr(j, "\"all_invariants_pass\":true") || std::strstr(j, "\"all_invariants_pass\": true"));
    };
    if (st != OFFSIM_OK || !pass(summary))
        std::fprintf(stderr, "executor summary (status %d): %.3000s\n", static_cast<int>(st),
                     summary ? summary : offsim_last_error());
    CHECK(st == OFFSIM_OK);
    CHECK(pass(summary));
    offsim_string_free(summary);
    offsim_scenario_free(s);
    return 0;
}

static int last_error_threads() {
    // the thread-local last error: concurrent failing calls on 8 threads
    // each see their own message
    std::vector<std::thread> th;
    std::vector<int> ok(8, 0);
    for (int t = 0; t < 8; ++t)
        th.emplace_back([t, &ok] {
            int good = 1;
            for (int i = 0; i < 200; ++i) {
                const fy_status s = fy_adamw_tune(t % 2 ? 2 : 0, 3, 0);  // both invalid
                const char* e = fy_last_error();
                good &= s == FY_ERR_CONFIG && e != nullptr &&
                        std::strstr(e, t % 2 ? "path must be" : "unroll must be") != nullptr;
            }
            ok[t] = good;
        });
    for (auto& x : th) x.join();
    for (int v : ok) CHECK(v == 1);
    CHECK(fy_adamw_tune(1, 3, 0) == FY_OK);
    return 0;
}

int main(int argc, char** argv) {
    const char* dir = argc > 1 ? argv[1] : "/tmp";
    if (int r = last_error_threads()) return r;
    if (int r = pipeline_case()) return r;
    if (int r = swap_case(dir)) return r;
    if (int r = executor_case(dir)) return r;
    std::printf("host pipeline driver: all checks passed\n");
    return 0;
}
