// xfer_microbench.cu — host-link microbenchmark for the zero-copy transfer
// design (not product code).  Gathers M random 256-B rows from a large pinned
// host table into HBM slots (and the reverse write-back), with variants:
//   load flavour (default / .nc / .cv), rows per group in flight, grid size,
//   random vs contiguous rows (GPU TLB reach over sysmem), and a
//   hugepage-backed registered allocation.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o xfer_mb xfer_microbench.cu
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
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

template <int MODE, int UNR>
__global__ void gather(const float4 *__restrict__ host, float4 *__restrict__ dev, const unsigned *rows,
                       const unsigned *slots, int M, int D4) {
    const int G = D4;  // lanes per row (D4 <= 32)
    const int gpb = blockDim.x / G, lane = threadIdx.x % G;
    const int ng = gridDim.x * gpb;
    for (int base = (blockIdx.x * gpb + threadIdx.x / G) * UNR; base < M; base += ng * UNR) {
        float4 v[UNR];
#pragma unroll
        for (int r = 0; r < UNR; r++) {
            int k = base + r;
            if (k < M) {
                const float4 *p = host + (size_t)rows[k] * D4 + lane;
                if (MODE == 0) v[r] = *p;
                else if (MODE == 1) v[r] = __ldg(p);
                else v[r] = __ldcv(p);
            }
        }
#pragma unroll
        for (int r = 0; r < UNR; r++) {
            int k = base + r;
            if (k < M) dev[(size_t)slots[k] * D4 + lane] = v[r];
        }
    }
}

__global__ void scatter_back(float4 *host, const float4 *dev, const unsigned *rows, const unsigned *slots,
                             int M, int D4) {
    const int G = D4;
    const int gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int k = blockIdx.x * gpb + threadIdx.x / G; k < M; k += gridDim.x * gpb)
        host[(size_t)rows[k] * D4 + lane] = dev[(size_t)slots[k] * D4 + lane];
}

int main(int argc, char **argv) {
    const size_t R = argc > 1 ? strtoull(argv[1], 0, 10) : 33000000ull;  // rows
    const int D = 64, D4 = D / 4;
    const int Ms[] = {1800, 6000, 60000};
    const size_t bytes = R * D * sizeof(float);
    float *h = nullptr;
    CK(cudaHostAlloc((void **)&h, bytes, cudaHostAllocMapped));
    memset(h, 0, bytes);
    // hugepage-backed registered alternative
    size_t hbytes = (bytes + (2u << 20) - 1) & ~((size_t)(2u << 20) - 1);
    float *hh = (float *)mmap(nullptr, hbytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(hh, hbytes, MADV_HUGEPAGE);
    memset(hh, 0, hbytes);
    bool reg_ok = cudaHostRegister(hh, hbytes, cudaHostRegisterMapped) == cudaSuccess;
    (void)cudaGetLastError();
    float4 *dev;
    CK(cudaMalloc(&dev, (size_t)4000000 * D * 4));
    unsigned *d_rows, *d_slots;
    CK(cudaMalloc(&d_rows, 60000 * 4));
    CK(cudaMalloc(&d_slots, 60000 * 4));
    std::mt19937_64 rng(1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto fn) {
        fn();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int it = 0; it < 10; it++) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        return best * 1000.f;  // us
    };
    for (int contiguous = 0; contiguous < 2; contiguous++) {
        for (int M : Ms) {
            std::vector<unsigned> rows(M), slots(M);
            size_t start = rng() % (R - M);
            for (int k = 0; k < M; k++) {
                rows[k] = contiguous ? (unsigned)(start + k) : (unsigned)(rng() % R);
                slots[k] = (unsigned)(rng() % 4000000);
            }
            CK(cudaMemcpy(d_rows, rows.data(), M * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d_slots, slots.data(), M * 4, cudaMemcpyHostToDevice));
            const double mb = (double)M * D * 4 / 1e6;
            for (int grid : {37, 148, 296, 592}) {
                float t0 = timeit([&] { gather<0, 4><<<grid, 256>>>((const float4 *)h, dev, d_rows, d_slots, M, D4); });
                float t1 = timeit([&] { gather<1, 4><<<grid, 256>>>((const float4 *)h, dev, d_rows, d_slots, M, D4); });
                float t2 = timeit([&] { gather<2, 4><<<grid, 256>>>((const float4 *)h, dev, d_rows, d_slots, M, D4); });
                float t3 = timeit([&] { gather<0, 1><<<grid, 256>>>((const float4 *)h, dev, d_rows, d_slots, M, D4); });
                float t4 = timeit([&] { scatter_back<<<grid, 256>>>((float4 *)h, dev, d_rows, d_slots, M, D4); });
                float t5 = reg_ok ? timeit([&] { gather<0, 4><<<grid, 256>>>((const float4 *)hh, dev, d_rows, d_slots, M, D4); }) : -1;
                printf("%s M=%6d grid=%3d | ld %.1fus (%.1f GB/s) | ldg %.1fus | ldcv %.1fus | ld unr1 %.1fus | "
                       "writeback %.1fus (%.1f GB/s) | hugepage-reg ld %.1fus\n",
                       contiguous ? "contig" : "random", M, grid, t0, mb / t0 * 1e-3 * 1e3, t1, t2, t3, t4,
                       mb / t4 * 1e-3 * 1e3, t5);
            }
        }
    }
    // copy-engine reference: one contiguous H2D of M rows
    for (int M : Ms) {
        float t = timeit([&] { cudaMemcpyAsync(dev, h, (size_t)M * D * 4, cudaMemcpyHostToDevice); });
        printf("memcpy H2D contiguous M=%d: %.1fus (%.1f GB/s)\n", M, t, (double)M * D * 4 / t / 1e3);
    }
    return 0;
}
