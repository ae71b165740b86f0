// GPU-side latency of the neighbour flag handshake (pwadv_signal_peers /
// pwadv_wait_peers) with ranks emulated as host threads on one GPU — in C++,
// so the host enqueues far ahead of the GPU (the Python threads of
// tools/handshake_cost.py are GIL-bound at 8 ranks).
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/handshake_latency.cu \
//        -Lpaper_2010_01545_b200 -lpwadv -Xlinker -rpath,'$ORIGIN/../paper_2010_01545_b200' \
//        -o tools/handshake_latency
//   tools/handshake_latency [px py rounds spin_us]
//
// Each rank's round: a one-thread spin kernel of spin_us (the "step"), then
// signal its neighbours (px x py periodic torus, as decomp.neighbour_ranks)
// and wait for them. The per-round time minus that of the same loop without
// the handshake is the handshake's critical-path cost on the GPU: flag write
// after the step (fenced), the neighbours' front ends observing it, and the
// next kernel launching behind the wait.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <thread>
#include <vector>

#include "../include/pwadv.h"

__global__ void spin(long long cycles)
{
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

static void ck(cudaError_t e, const char *w)
{
    if (e != cudaSuccess) {
        fprintf(stderr, "%s: %s\n", w, cudaGetErrorString(e));
        exit(1);
    }
}

static void ckp(int rc, const char *w)
{
    if (rc) {
        fprintf(stderr, "%s: %s\n", w, pwadv_last_error());
        exit(1);
    }
}

int main(int argc, char **argv)
{
    const int px = argc > 1 ? atoi(argv[1]) : 2, py = argc > 2 ? atoi(argv[2]) : 4;
    const int rounds = argc > 3 ? atoi(argv[3]) : 2000;
    const double spin_us = argc > 4 ? atof(argv[4]) : 20.0;
    const int n = px * py;
    int clk_khz = 0;
    ck(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0), "clock");
    const long long cycles = (long long)(spin_us * clk_khz / 1e3);
    std::vector<uint64_t *> flags(n);
    for (int r = 0; r < n; ++r) {
        ck(cudaMalloc(&flags[r], n * sizeof(uint64_t)), "malloc");
        ck(cudaMemset(flags[r], 0, n * sizeof(uint64_t)), "memset");
    }
    std::vector<std::vector<int>> nbrs(n);
    for (int r = 0; r < n; ++r) {
        const int cx = r / py, cy = r % py;
        std::set<int> s;
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy) {
                if (!dx && !dy) continue;
                const int q = ((cx + dx + px) % px) * py + (cy + dy + py) % py;
                if (q != r) s.insert(q);
            }
        nbrs[r].assign(s.begin(), s.end());
    }
    int *err = nullptr;
    ck(cudaMalloc(&err, sizeof(int)), "malloc err");
    ck(cudaMemset(err, 0, sizeof(int)), "memset err");
    ck(cudaDeviceSynchronize(), "sync");
    const int only = getenv("HS_MODE") ? atoi(getenv("HS_MODE")) : -1;
    const unsigned long long tmo = getenv("HS_TIMEOUT_NS") ? strtoull(getenv("HS_TIMEOUT_NS"), 0, 10) : 0;
    for (int mode = 0; mode < 4; ++mode) {
        if (only >= 0 && mode != only && mode != 0) continue;  // 0: spin only, 1: signal + wait calls, 2: one batch, 3: kernel
        std::vector<double> per(n);
        std::vector<std::thread> ts;
        // fresh flags per mode (values restart at 1)
        for (int r = 0; r < n; ++r) ck(cudaMemset(flags[r], 0, n * sizeof(uint64_t)), "memset");
        ck(cudaDeviceSynchronize(), "sync");
        const uint64_t base = 0;
        for (int r = 0; r < n; ++r)
            ts.emplace_back([&, r] {
                cudaStream_t s;
                ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
                std::vector<uint64_t *> sig, wt;
                for (int q : nbrs[r]) {
                    sig.push_back(flags[q] + r);
                    wt.push_back(flags[r] + q);
                }
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                for (int k = 0; k < 20; ++k) spin<<<1, 1, 0, s>>>(cycles);
                ck(cudaStreamSynchronize(s), "warm");
                cudaEventRecord(a, s);
                for (int k = 1; k <= rounds; ++k) {
                    spin<<<1, 1, 0, s>>>(cycles);
                    if (mode == 1) {
                        ckp(pwadv_signal_peers(sig.data(), (int)sig.size(), base + k, s), "signal");
                        ckp(pwadv_wait_peers(wt.data(), (int)wt.size(), base + k, s), "wait");
                    } else if (mode == 2) {
                        ckp(pwadv_handshake(sig.data(), (int)sig.size(), wt.data(), (int)wt.size(),
                                            base + k, s), "handshake");
                    } else if (mode == 3) {
                        ckp(pwadv_handshake_kernel(sig.data(), (int)sig.size(), wt.data(), (int)wt.size(),
                                                   base + k, err, tmo, s), "handshake kernel");
                    }
                }
                cudaEventRecord(b, s);
                ck(cudaStreamSynchronize(s), "run");
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                per[r] = ms * 1e3 / rounds;
                cudaStreamDestroy(s);
            });
        for (auto &t : ts) t.join();
        const double worst = *std::max_element(per.begin(), per.end());
        printf("{\"what\": \"handshake latency (C++ threads, one GPU)\", \"decomposition\": \"%dx%d\", "
               "\"neighbours\": %zu, \"handshake\": \"%s\", \"spin_us\": %.1f, \"us_per_round\": %.2f}\n",
               px, py, nbrs[0].size(), mode == 0 ? "none" : mode == 1 ? "signal+wait" : mode == 2 ? "one batch" : "kernel",
               spin_us, worst);
        fflush(stdout);
    }
    int herr = 0;
    ck(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost), "err");
    if (herr) printf("{\"error\": \"handshake kernel timed out\"}\n");
    return 0;
}
