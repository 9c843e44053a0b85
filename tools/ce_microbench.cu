// ce_microbench.cu — copy-engine alternatives for the scratchpad transfer
// (not product code):
//   (1) cudaMemcpyBatchAsync of M random 256-B host rows -> device slots, and
//       device slots -> random host rows (one descriptor per row);
//   (2) CPU threads gather M random rows into a pinned staging buffer, then
//       one contiguous H2D DMA (and the reverse for write-backs);
// each alone and next to the HBM gather kernel (interference).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ce_mb ce_microbench.cu -lpthread
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

__global__ void gather_rows(const float4 *__restrict__ st, const unsigned *__restrict__ idx, float4 *out,
                            int nrows, int D4) {
    const int G = D4, gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int r = blockIdx.x * gpb + threadIdx.x / G; r < nrows; r += gridDim.x * gpb)
        out[(size_t)r * D4 + lane] = __ldg(st + (size_t)idx[r] * D4 + lane);
}

__global__ void scatter_rows(const float4 *__restrict__ in, const unsigned *__restrict__ slots, float4 *st,
                             int nrows, int D4) {
    const int G = D4, gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int r = blockIdx.x * gpb + threadIdx.x / G; r < nrows; r += gridDim.x * gpb)
        st[(size_t)slots[r] * D4 + lane] = in[(size_t)r * D4 + lane];
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const int D = 64, D4 = 16, RB = D * 4;
    const size_t R = 33000000, S = 3400000;
    float *h;
    CK(cudaHostAlloc((void **)&h, R * D * 4, cudaHostAllocMapped));
    memset(h, 1, R * D * 4);
    float4 *st;
    CK(cudaMalloc(&st, S * D * 4));
    std::mt19937_64 rng(5);
    const int NR = 53248;
    std::vector<unsigned> gi(NR);
    for (auto &x : gi) x = rng() % S;
    unsigned *d_gi;
    float4 *gout;
    CK(cudaMalloc(&d_gi, NR * 4));
    CK(cudaMalloc(&gout, (size_t)NR * RB));
    CK(cudaMemcpy(d_gi, gi.data(), NR * 4, cudaMemcpyHostToDevice));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t a, b, c, d;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c); cudaEventCreate(&d);
    for (int M : {1800, 6000}) {
        std::vector<unsigned> rows(M), slots(M);
        for (int k = 0; k < M; k++) { rows[k] = rng() % R; slots[k] = rng() % S; }
        std::vector<void *> dst(M), src(M), wdst(M), wsrc(M);
        std::vector<size_t> sz(M, RB), idx0(1, 0);
        for (int k = 0; k < M; k++) {
            dst[k] = (char *)st + (size_t)slots[k] * RB;
            src[k] = (char *)h + (size_t)rows[k] * RB;
            wdst[k] = (char *)h + (size_t)((rows[k] + 7777) % R) * RB;
            wsrc[k] = (char *)st + (size_t)((slots[k] + 99) % S) * RB;
        }
        cudaMemcpyAttributes at{};
        at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        at.flags = cudaMemcpyFlagPreferOverlapWithCompute;
        size_t fail = 0;
        // (1) batch memcpy
        for (int it = 0; it < 3; it++) {
            CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), M, &at, idx0.data(), 1, &fail, s1));
            CK(cudaStreamSynchronize(s1));
        }
        double t_api = 0;
        float best_h2d = 1e9, best_d2h = 1e9;
        for (int it = 0; it < 10; it++) {
            double t0 = now_us();
            cudaEventRecord(a, s1);
            CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), M, &at, idx0.data(), 1, &fail, s1));
            cudaEventRecord(b, s1);
            t_api += now_us() - t0;
            CK(cudaMemcpyBatchAsync(wdst.data(), wsrc.data(), sz.data(), M, &at, idx0.data(), 1, &fail, s1));
            cudaEventRecord(c, s1);
            CK(cudaEventSynchronize(c));
            float m1, m2;
            cudaEventElapsedTime(&m1, a, b);
            cudaEventElapsedTime(&m2, b, c);
            best_h2d = std::min(best_h2d, m1 * 1000.f);
            best_d2h = std::min(best_d2h, m2 * 1000.f);
        }
        printf("batchmemcpy M=%d: H2D %.1f us, D2H %.1f us, API call %.1f us (host)\n", M, best_h2d, best_d2h, t_api / 10);
        // interference: gather kernel next to repeated batch copies
        {
            float alone = 0, with = 0;
            for (int it = 0; it < 20; it++) {
                cudaEventRecord(a, s0);
                gather_rows<<<1184, 256, 0, s0>>>(st, d_gi, gout, NR, D4);
                cudaEventRecord(b, s0);
                CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b); alone += ms;
            }
            for (int it = 0; it < 20; it++) {
                CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), M, &at, idx0.data(), 1, &fail, s1));
                CK(cudaMemcpyBatchAsync(wdst.data(), wsrc.data(), sz.data(), M, &at, idx0.data(), 1, &fail, s1));
                cudaEventRecord(a, s0);
                gather_rows<<<1184, 256, 0, s0>>>(st, d_gi, gout, NR, D4);
                cudaEventRecord(b, s0);
                CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b); with += ms;
                CK(cudaStreamSynchronize(s1));
            }
            printf("  gather kernel alone %.1f us, with batch-memcpy traffic %.1f us\n", alone * 50, with * 50);
        }
        // (2) CPU gather into pinned staging + one DMA + scatter kernel
        float *stage;
        CK(cudaHostAlloc((void **)&stage, (size_t)M * RB, 0));
        float4 *dstage;
        unsigned *d_slots;
        CK(cudaMalloc(&dstage, (size_t)M * RB));
        CK(cudaMalloc(&d_slots, M * 4));
        CK(cudaMemcpy(d_slots, slots.data(), M * 4, cudaMemcpyHostToDevice));
        for (int nt : {1, 4, 8}) {
            double best = 1e9;
            for (int it = 0; it < 10; it++) {
                double t0 = now_us();
                std::vector<std::thread> th;
                for (int k = 0; k < nt; k++)
                    th.emplace_back([&, k] {
                        for (int r = k; r < M; r += nt)
                            memcpy((char *)stage + (size_t)r * RB, (char *)h + (size_t)rows[r] * RB, RB);
                    });
                for (auto &x : th) x.join();
                double t1 = now_us();
                best = std::min(best, t1 - t0);
            }
            printf("  CPU gather M=%d threads=%d: %.1f us (incl. thread spawn)\n", M, nt, best);
        }
        float best_dma = 1e9;
        for (int it = 0; it < 10; it++) {
            cudaEventRecord(a, s1);
            CK(cudaMemcpyAsync(dstage, stage, (size_t)M * RB, cudaMemcpyHostToDevice, s1));
            scatter_rows<<<148, 256, 0, s1>>>(dstage, d_slots, st, M, D4);
            cudaEventRecord(b, s1);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            best_dma = std::min(best_dma, ms * 1000.f);
        }
        printf("  staged H2D DMA + scatter kernel M=%d: %.1f us\n", M, best_dma);
        cudaFreeHost(stage);
        cudaFree(dstage);
        cudaFree(d_slots);
    }
    return 0;
}
