// tma_xfer_microbench.cu — host-link row exchange through TMA bulk copies
// (cp.async.bulk) vs plain SM zero-copy loads/stores (not product code).
//
// Question: can the GPU do BOTH directions of [Collect]/[Insert] itself
// (victim write-back HBM -> host row, missed row host -> HBM slot) at the
// host-link rate without slowing the concurrent HBM-bound Train kernels?
// Plain 16-B zero-copy stores from >= 4 CTAs slowed a concurrent HBM gather
// ~6x (profiles/r01_interference_microbench.txt).  A bulk copy moves a whole
// 256-B row per request from one issuing thread.
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_mb tma_xfer_microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <algorithm>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// global (device or mapped host) -> shared
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// shared -> global (device or mapped host)
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void gather_rows(const float4 *__restrict__ st, const unsigned *__restrict__ idx, float4 *out,
                            int nrows, int D4) {
    const int G = D4, gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int r = blockIdx.x * gpb + threadIdx.x / G; r < nrows; r += gridDim.x * gpb)
        out[(size_t)r * D4 + lane] = __ldg(st + (size_t)idx[r] * D4 + lane);
}

// MODE 0 exchange (write-back + pull), 1 pull only, 2 write-back only.
// Plain SM path: 16 lanes x float4 per row.
template <int MODE>
__global__ void plain_xchg(float *host, float *dev, const unsigned *rows, const unsigned *old_rows,
                           const unsigned *slots, int M, int D) {
    const int D4 = D / 4, G = D4, gpb = blockDim.x / G, lane = threadIdx.x % G;
    float4 *h = (float4 *)host, *d = (float4 *)dev;
    for (int k = blockIdx.x * gpb + threadIdx.x / G; k < M; k += gridDim.x * gpb) {
        float4 x;
        if (MODE != 2) x = __ldcv(h + (size_t)rows[k] * D4 + lane);
        if (MODE != 1) h[(size_t)old_rows[k] * D4 + lane] = d[(size_t)slots[k] * D4 + lane];
        if (MODE != 2) d[(size_t)slots[k] * D4 + lane] = x;
    }
}

// TMA path: one CTA of 32 threads per "engine"; each round stages NB rows:
// lane i < NB issues the bulk loads of rows i (victim from HBM, new row from
// host) onto one mbarrier; after the wait, lanes issue the bulk stores
// (victim -> host row, new row -> HBM slot).  Two stages ping-pong so the
// loads of round r+1 fly while round r is stored.
template <int MODE, int NB>
__global__ void __launch_bounds__(32) tma_xchg(float *host, float *dev, const unsigned *rows,
                                               const unsigned *old_rows, const unsigned *slots, int M, int D) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[2];
    const uint32_t rowb = D * 4;
    unsigned char *vic = sm;                       // [2][NB][rowb]
    unsigned char *nw = sm + 2 * NB * rowb;        // [2][NB][rowb]
    const int lane = threadIdx.x;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int per = NB;
    const int nround = (M + per - 1) / per;
    uint32_t phase[2] = {0, 0};
    auto issue = [&](int r, int st) {
        const int k0 = r * per;
        const int cnt = min(per, M - k0);
        const uint32_t bytes = (uint32_t)cnt * rowb * ((MODE == 0) ? 2 : 1);
        if (lane == 0) mbar_expect_tx(&bar[st], bytes);
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) {
            const int k = k0 + i;
            if (MODE != 1) bulk_g2s(vic + ((size_t)st * NB + i) * rowb, dev + (size_t)slots[k] * D, rowb, &bar[st]);
            if (MODE != 2) bulk_g2s(nw + ((size_t)st * NB + i) * rowb, host + (size_t)rows[k] * D, rowb, &bar[st]);
        }
    };
    int r = blockIdx.x;
    if (r < nround) issue(r, 0);
    int st = 0;
    for (; r < nround; r += gridDim.x) {
        const int rn = r + gridDim.x;
        // stage st^1 is free once its stores have read smem
        if (rn < nround) {
            bulk_wait_read0();  // per thread: each lane waits for its own bulk groups
            __syncwarp();
            issue(rn, st ^ 1);
        }
        mbar_wait(&bar[st], phase[st]);
        phase[st] ^= 1;
        const int k0 = r * per;
        const int cnt = min(per, M - k0);
        for (int i = lane; i < cnt; i += 32) {
            const int k = k0 + i;
            if (MODE != 1) bulk_s2g(host + (size_t)old_rows[k] * D, vic + ((size_t)st * NB + i) * rowb, rowb);
            if (MODE != 2) bulk_s2g(dev + (size_t)slots[k] * D, nw + ((size_t)st * NB + i) * rowb, rowb);
        }
        bulk_commit();
        st ^= 1;
    }
    bulk_wait0();
}


// Deep-queue TMA: NS stages of NB rows per CTA (one warp); stage s is
// refilled with round r+NS as soon as the stores issued from it at round r
// have read shared memory (wait_group.read NS-1 keeps the newer ones going).
template <int MODE, int NB, int NS>
__global__ void __launch_bounds__(32) tma_deep(float *host, float *dev, const unsigned *rows,
                                               const unsigned *old_rows, const unsigned *slots, int M, int D) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NS];
    const uint32_t rowb = D * 4;
    const int lane = threadIdx.x;
    constexpr int W = (MODE == 0) ? 2 : 1;
    if (lane == 0) {
        for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // this CTA's contiguous share of rows, in rounds of NB
    const int per_cta = (M + gridDim.x - 1) / gridDim.x;
    const int k_lo = blockIdx.x * per_cta, k_hi = min(M, k_lo + per_cta);
    const int nround = k_hi > k_lo ? (k_hi - k_lo + NB - 1) / NB : 0;
    auto buf = [&](int s, int i, int w) { return sm + (((size_t)s * NB + i) * W + w) * rowb; };
    auto issue = [&](int r) {
        const int s = r % NS, k0 = k_lo + r * NB, cnt = min(NB, k_hi - k0);
        if (lane == 0) mbar_expect_tx(&bar[s], (uint32_t)cnt * rowb * W);
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) {
            const int k = k0 + i;
            if (MODE != 1) bulk_g2s(buf(s, i, 0), dev + (size_t)slots[k] * D, rowb, &bar[s]);
            if (MODE != 2) bulk_g2s(buf(s, i, W - 1), host + (size_t)rows[k] * D, rowb, &bar[s]);
        }
    };
    for (int r = 0; r < min(NS, nround); r++) issue(r);
    for (int r = 0; r < nround; r++) {
        const int s = r % NS, k0 = k_lo + r * NB, cnt = min(NB, k_hi - k0);
        mbar_wait(&bar[s], (uint32_t)((r / NS) & 1));
        for (int i = lane; i < cnt; i += 32) {
            const int k = k0 + i;
            if (MODE != 1) bulk_s2g(host + (size_t)old_rows[k] * D, buf(s, i, 0), rowb);
            if (MODE != 2) bulk_s2g(dev + (size_t)slots[k] * D, buf(s, i, W - 1), rowb);
        }
        bulk_commit();
        if (r + NS < nround) {
            bulk_wait_read0();
            __syncwarp();
            issue(r + NS);
        }
    }
    bulk_wait0();
}

int main() {
    const int D = 64, D4 = 16;
    const size_t R = 33000000, S = 3400000;
    const int NR = 53248;
    float *h;
    CK(cudaHostAlloc((void **)&h, R * D * 4, cudaHostAllocMapped));
    float *dev;
    float4 *out;
    CK(cudaMalloc(&dev, S * D * 4));
    CK(cudaMalloc(&out, (size_t)NR * D * 4));
    std::mt19937_64 rng(3);
    std::vector<unsigned> gi(NR);
    for (auto &x : gi) x = rng() % S;
    unsigned *d_gi;
    CK(cudaMalloc(&d_gi, NR * 4));
    CK(cudaMemcpy(d_gi, gi.data(), NR * 4, cudaMemcpyHostToDevice));
    const int MMAX = 60000;
    std::vector<unsigned> rows(MMAX), old(MMAX), slots(MMAX);
    for (int k = 0; k < MMAX; k++) {
        rows[k] = rng() % (R / 2);
        old[k] = R / 2 + rng() % (R / 2);
        slots[k] = rng() % S;
    }
    unsigned *d_rows, *d_old, *d_slots;
    CK(cudaMalloc(&d_rows, MMAX * 4));
    CK(cudaMalloc(&d_old, MMAX * 4));
    CK(cudaMalloc(&d_slots, MMAX * 4));
    CK(cudaMemcpy(d_rows, rows.data(), MMAX * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_old, old.data(), MMAX * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_slots, slots.data(), MMAX * 4, cudaMemcpyHostToDevice));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = 2 * 2 * 32 * D * 4;  // NB=32
    CK(cudaFuncSetAttribute(tma_xchg<0, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(tma_xchg<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(tma_xchg<2, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto time_gather = [&](int reps) {
        float tot = 0;
        for (int i = 0; i < reps; i++) {
            cudaEventRecord(a, s0);
            gather_rows<<<1184, 256, 0, s0>>>((const float4 *)dev, d_gi, out, NR, D4);
            cudaEventRecord(b, s0);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            tot += ms;
        }
        return tot / reps * 1000.f;
    };
    // kind: 0 plain (grid CTAs x 256 thr), 1 tma (grid CTAs x 32 thr)
    auto launch = [&](int kind, int mode, int grid, int M, cudaStream_t s) {
        if (kind == 0) {
            if (mode == 0) plain_xchg<0><<<grid, 256, 0, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
            if (mode == 1) plain_xchg<1><<<grid, 256, 0, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
            if (mode == 2) plain_xchg<2><<<grid, 256, 0, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
        } else {
            if (mode == 0) tma_xchg<0, 32><<<grid, 32, smem, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
            if (mode == 1) tma_xchg<1, 32><<<grid, 32, smem, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
            if (mode == 2) tma_xchg<2, 32><<<grid, 32, smem, s>>>(h, dev, d_rows, d_old, d_slots, M, D);
        }
    };
    auto time_alone = [&](int kind, int mode, int grid, int M) {
        for (int i = 0; i < 3; i++) launch(kind, mode, grid, M, s1);
        cudaEventRecord(a, s1);
        const int reps = 10;
        for (int i = 0; i < reps; i++) launch(kind, mode, grid, M, s1);
        cudaEventRecord(b, s1);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms * 1000.f / reps;
    };
    // correctness spot check of the TMA exchange: pull rows -> slots
    {
        std::vector<float> hv(D);
        CK(cudaMemset(dev, 0, S * D * 4));
        for (int k = 0; k < 64; k++)
            for (int c = 0; c < D; c++) h[(size_t)rows[k] * D + c] = (float)(k * 1000 + c);
        launch(1, 1, 2, 64, s1);
        CK(cudaStreamSynchronize(s1));
        int bad = 0;
        for (int k = 0; k < 64; k++) {
            CK(cudaMemcpy(hv.data(), dev + (size_t)slots[k] * D, D * 4, cudaMemcpyDeviceToHost));
            for (int c = 0; c < D; c++) bad += hv[c] != (float)(k * 1000 + c);
        }
        // write-back: slots -> old rows
        launch(1, 2, 2, 64, s1);
        CK(cudaStreamSynchronize(s1));
        for (int k = 0; k < 64; k++)
            for (int c = 0; c < D; c++) bad += h[(size_t)old[k] * D + c] != (float)(k * 1000 + c);
        printf("tma correctness: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
    }
    const char *mname[3] = {"exchange", "pull", "writeback"};
#define SETSM(NB, NS)                                                                                 \
    CK(cudaFuncSetAttribute(tma_deep<0, NB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * NS * 2 * D * 4)); \
    CK(cudaFuncSetAttribute(tma_deep<1, NB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * NS * 2 * D * 4)); \
    CK(cudaFuncSetAttribute(tma_deep<2, NB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * NS * 2 * D * 4));
    SETSM(32, 4) SETSM(64, 4) SETSM(32, 8) SETSM(64, 6)
    auto launch_deep = [&](int cfg, int mode, int grid, int M, cudaStream_t s) {
#define LD(NB, NS)                                                                                       \
    {                                                                                                    \
        const size_t sb = (size_t)NB * NS * (mode == 0 ? 2 : 1) * D * 4;                                 \
        if (mode == 0) tma_deep<0, NB, NS><<<grid, 32, sb, s>>>(h, dev, d_rows, d_old, d_slots, M, D);  \
        if (mode == 1) tma_deep<1, NB, NS><<<grid, 32, sb, s>>>(h, dev, d_rows, d_old, d_slots, M, D);  \
        if (mode == 2) tma_deep<2, NB, NS><<<grid, 32, sb, s>>>(h, dev, d_rows, d_old, d_slots, M, D);  \
    }
        if (cfg == 0) LD(32, 4)
        if (cfg == 1) LD(64, 4)
        if (cfg == 2) LD(32, 8)
        if (cfg == 3) LD(64, 6)
    };
    const char *cname[4] = {"NB32xNS4", "NB64xNS4", "NB32xNS8", "NB64xNS6"};
    auto time_deep = [&](int cfg, int mode, int grid, int M) {
        for (int i = 0; i < 3; i++) launch_deep(cfg, mode, grid, M, s1);
        cudaEventRecord(a, s1);
        for (int i = 0; i < 10; i++) launch_deep(cfg, mode, grid, M, s1);
        cudaEventRecord(b, s1);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms * 100.f;
    };
    // correctness of the deep kernel (exchange): rows -> slots, slots -> old rows
    {
        int bad = 0;
        CK(cudaMemset(dev, 0, S * D * 4));
        for (int k = 0; k < 300; k++)
            for (int c = 0; c < D; c++) h[(size_t)rows[k] * D + c] = (float)(k * 1000 + c);
        launch_deep(1, 1, 3, 300, s1);
        launch_deep(1, 2, 3, 300, s1);
        CK(cudaStreamSynchronize(s1));
        for (int k = 0; k < 300; k++)
            for (int c = 0; c < D; c++) bad += h[(size_t)old[k] * D + c] != (float)(k * 1000 + c);
        printf("tma_deep correctness: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
    }
    time_gather(5);
    const float g0 = time_gather(50);
    printf("gather alone: %.1f us\n", g0);
    for (int M : {1800, 6000}) {
        for (int cfg = 0; cfg < 4; cfg++) {
            for (int grid : {2, 4, 8, 16}) {
                printf("%s M=%5d grid=%3d |", cname[cfg], M, grid);
                for (int mode = 0; mode < 3; mode++) {
                    const float us = time_deep(cfg, mode, grid, M);
                    const double bytes = (double)M * D * 4 * (mode == 0 ? 2 : 1);
                    const int nbg = (int)std::min(2000.f, std::max(20.f, 4000.f / us));
                    for (int i = 0; i < nbg; i++) launch_deep(cfg, mode, grid, M, s1);
                    const float gi_us = time_gather(20);
                    CK(cudaDeviceSynchronize());
                    printf(" %s %7.1fus %5.1fGB/s gather x%.2f |", mname[mode], us, bytes / (us * 1e-6) / 1e9,
                           gi_us / g0);
                }
                printf("\n");
            }
        }
    }
    // the previous plain / 2-stage sweep, M=1800 only, for the same-box comparison
    for (int M : {1800}) {
        for (int kind = 0; kind < 2; kind++) {
            for (int grid : {8, 16, 37}) {
                printf("%-5s M=%5d grid=%3d |", kind ? "tma2" : "plain", M, grid);
                for (int mode = 0; mode < 3; mode++) {
                    const float us = time_alone(kind, mode, grid, M);
                    const double bytes = (double)M * D * 4 * (mode == 0 ? 2 : 1);
                    const int nbg = (int)std::min(2000.f, std::max(20.f, 4000.f / us));
                    for (int i = 0; i < nbg; i++) launch(kind, mode, grid, M, s1);
                    const float gi_us = time_gather(20);
                    CK(cudaDeviceSynchronize());
                    printf(" %s %7.1fus %5.1fGB/s gather x%.2f |", mname[mode], us, bytes / (us * 1e-6) / 1e9,
                           gi_us / g0);
                }
                printf("\n");
            }
        }
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
