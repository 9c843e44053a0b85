// interference_microbench.cu — does host-link traffic slow HBM-bound kernels?
// (not product code).  Times a 27 MB HBM gather-like kernel (the k_fwd
// shape: random 256-B rows -> contiguous output) alone and while another
// stream runs (a) SM zero-copy exchange of random host rows, (b) copy-engine
// H2D + D2H DMA of contiguous pinned buffers.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o interf_mb interference_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
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

// MODE 0: write-back + pull, 1: pull only (PCIe reads), 2: write-back only (PCIe writes)
template <int MODE>
__global__ void exchange(float4 *host, float4 *dev, const unsigned *rows, const unsigned *old_rows,
                         const unsigned *slots, int M, int D4, int reps) {
    const int G = D4, gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int rep = 0; rep < reps; rep++)
        for (int k = blockIdx.x * gpb + threadIdx.x / G; k < M; k += gridDim.x * gpb) {
            if (MODE != 1) {
                float4 v = dev[(size_t)slots[k] * D4 + lane];
                host[(size_t)old_rows[k] * D4 + lane] = v;
            }
            if (MODE != 2) {
                float4 x = __ldcv(host + (size_t)rows[k] * D4 + lane);
                dev[(size_t)slots[k] * D4 + lane] = x;
            }
        }
}

int main() {
    const int D = 64, D4 = 16;
    const size_t R = 33000000, S = 3400000;
    const int NR = 53248;  // rows gathered per "forward"
    float *h;
    CK(cudaHostAlloc((void **)&h, R * D * 4, cudaHostAllocMapped));
    float4 *st, *out;
    CK(cudaMalloc(&st, S * D * 4));
    CK(cudaMalloc(&out, (size_t)NR * D * 4));
    std::mt19937_64 rng(3);
    std::vector<unsigned> gi(NR);
    for (auto &x : gi) x = rng() % S;
    unsigned *d_gi;
    CK(cudaMalloc(&d_gi, NR * 4));
    CK(cudaMemcpy(d_gi, gi.data(), NR * 4, cudaMemcpyHostToDevice));
    const int M = 1800 * 3;
    std::vector<unsigned> rows(M), old(M), slots(M);
    for (int k = 0; k < M; k++) {
        rows[k] = rng() % (R / 2);
        old[k] = R / 2 + rng() % (R / 2);
        slots[k] = rng() % S;
    }
    unsigned *d_rows, *d_old, *d_slots;
    CK(cudaMalloc(&d_rows, M * 4));
    CK(cudaMalloc(&d_old, M * 4));
    CK(cudaMalloc(&d_slots, M * 4));
    CK(cudaMemcpy(d_rows, rows.data(), M * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_old, old.data(), M * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_slots, slots.data(), M * 4, cudaMemcpyHostToDevice));
    // DMA buffers
    const size_t dbytes = 64 << 20;
    void *hd, *hd2, *dd, *dd2;
    CK(cudaHostAlloc(&hd, dbytes, 0));
    CK(cudaHostAlloc(&hd2, dbytes, 0));
    CK(cudaMalloc(&dd, dbytes));
    CK(cudaMalloc(&dd2, dbytes));
    cudaStream_t s0, s1, s2;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time_gather = [&](int reps) {
        float tot = 0;
        for (int i = 0; i < reps; i++) {
            cudaEventRecord(a, s0);
            gather_rows<<<1184, 256, 0, s0>>>(st, d_gi, out, NR, D4);
            cudaEventRecord(b, s0);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            tot += ms;
        }
        return tot / reps * 1000.f;
    };
    time_gather(5);
    printf("gather alone: %.1f us\n", time_gather(50));
    for (int grid : {4, 16, 37, 148}) {
        exchange<0><<<grid, 256, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 100);
        float t0 = time_gather(30);
        CK(cudaDeviceSynchronize());
        exchange<1><<<grid, 256, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 100);
        float t1 = time_gather(30);
        CK(cudaDeviceSynchronize());
        exchange<2><<<grid, 256, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 100);
        float t2 = time_gather(30);
        CK(cudaDeviceSynchronize());
        // throughput of each mode alone at this grid
        cudaEventRecord(a, s1);
        exchange<1><<<grid, 256, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 10);
        cudaEventRecord(b, s1);
        CK(cudaEventSynchronize(b));
        float mr; cudaEventElapsedTime(&mr, a, b);
        cudaEventRecord(a, s1);
        exchange<2><<<grid, 256, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 10);
        cudaEventRecord(b, s1);
        CK(cudaEventSynchronize(b));
        float mw; cudaEventElapsedTime(&mw, a, b);
        printf("grid %3d: gather next to exchange %.1f us | next to pulls only %.1f us | next to write-backs only %.1f us"
               " || pulls alone %.1f GB/s, write-backs alone %.1f GB/s\n", grid, t0, t1, t2,
               10.0 * M * 256 / (mr * 1e-3) / 1e9, 10.0 * M * 256 / (mw * 1e-3) / 1e9);
    }
    for (int thr : {32, 64, 128, 256}) {
        exchange<2><<<1, thr, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 20);
        float t2 = time_gather(20);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a, s1);
        exchange<2><<<1, thr, 0, s1>>>((float4 *)h, st, d_rows, d_old, d_slots, M, D4, 4);
        cudaEventRecord(b, s1);
        CK(cudaEventSynchronize(b));
        float mw; cudaEventElapsedTime(&mw, a, b);
        printf("1 CTA x %3d threads write-backs: gather %.1f us, write-back rate %.1f GB/s\n", thr, t2,
               4.0 * M * 256 / (mw * 1e-3) / 1e9);
    }
    for (size_t chunk : {(size_t)512 << 10, (size_t)4 << 20}) {
        for (int k = 0; k < 400; k++) cudaMemcpyAsync(hd2, dd2, chunk, cudaMemcpyDeviceToHost, s2);
        float t = time_gather(30);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a, s2);
        for (int k = 0; k < 20; k++) cudaMemcpyAsync(hd2, dd2, chunk, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(b, s2);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("DMA D2H %zu KB back-to-back: gather %.1f us, D2H rate %.1f GB/s\n", chunk >> 10, t, 20.0 * chunk / (ms * 1e-3) / 1e9);
        for (int k = 0; k < 400; k++) cudaMemcpyAsync(dd, hd, chunk, cudaMemcpyHostToDevice, s1);
        t = time_gather(30);
        CK(cudaDeviceSynchronize());
        printf("DMA H2D %zu KB back-to-back: gather %.1f us\n", chunk >> 10, t);
    }
    for (int k = 0; k < 40; k++) {
        cudaMemcpyAsync(dd, hd, dbytes, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(hd2, dd2, dbytes, cudaMemcpyDeviceToHost, s2);
    }
    printf("gather with DMA H2D+D2H: %.1f us\n", time_gather(50));
    CK(cudaDeviceSynchronize());
    return 0;
}
