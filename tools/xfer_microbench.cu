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

// both directions per slot: write back the victim row, pull the missed row
// ORDER 0: ld dev v; st host v; ld host x; st dev x      (v1 kernel)
// ORDER 1: ld host x; ld dev v; st host v; st dev x      (all loads first, per row)
// ORDER 2: like 1 but all write-back stores of the UNR rows before any fill store
// ORDER 3: split roles: even groups write back, odd groups pull (slot read
//          ordering handled by a separate pass in the product; here timing only)
template <int ORDER, int UNR>
__global__ void exchange(float4 *host, float4 *dev, const unsigned *rows, const unsigned *old_rows,
                         const unsigned *slots, int M, int D4) {
    const int G = D4;
    const int gpb = blockDim.x / G, lane = threadIdx.x % G;
    const int ng = gridDim.x * gpb;
    int gid = blockIdx.x * gpb + threadIdx.x / G;
    if (ORDER == 3) {
        const bool wbrole = gid & 1;
        gid >>= 1;
        for (int k = gid; k < M; k += ng / 2) {
            if (wbrole) host[(size_t)old_rows[k] * D4 + lane] = dev[(size_t)slots[k] * D4 + lane];
            else dev[(size_t)slots[k] * D4 + lane] = host[(size_t)rows[k] * D4 + lane];
        }
        return;
    }
    for (int base = gid * UNR; base < M; base += ng * UNR) {
        float4 v[UNR], x[UNR];
        if (ORDER == 0) {
#pragma unroll
            for (int r = 0; r < UNR; r++) if (base + r < M) v[r] = dev[(size_t)slots[base + r] * D4 + lane];
#pragma unroll
            for (int r = 0; r < UNR; r++) if (base + r < M) host[(size_t)old_rows[base + r] * D4 + lane] = v[r];
#pragma unroll
            for (int r = 0; r < UNR; r++) if (base + r < M) x[r] = __ldcv(host + (size_t)rows[base + r] * D4 + lane);
#pragma unroll
            for (int r = 0; r < UNR; r++) if (base + r < M) dev[(size_t)slots[base + r] * D4 + lane] = x[r];
        } else {
#pragma unroll
            for (int r = 0; r < UNR; r++)
                if (base + r < M) {
                    x[r] = __ldcv(host + (size_t)rows[base + r] * D4 + lane);
                    v[r] = dev[(size_t)slots[base + r] * D4 + lane];
                }
            if (ORDER == 1) {
#pragma unroll
                for (int r = 0; r < UNR; r++)
                    if (base + r < M) {
                        host[(size_t)old_rows[base + r] * D4 + lane] = v[r];
                        dev[(size_t)slots[base + r] * D4 + lane] = x[r];
                    }
            } else {
#pragma unroll
                for (int r = 0; r < UNR; r++) if (base + r < M) host[(size_t)old_rows[base + r] * D4 + lane] = v[r];
#pragma unroll
                for (int r = 0; r < UNR; r++) if (base + r < M) dev[(size_t)slots[base + r] * D4 + lane] = x[r];
            }
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
    // combined exchange variants (random rows, disjoint read / write-back sets)
    unsigned *d_old;
    CK(cudaMalloc(&d_old, 60000 * 4));
    for (int M : Ms) {
        std::vector<unsigned> rows(M), old(M), slots(M);
        for (int k = 0; k < M; k++) {
            rows[k] = (unsigned)(rng() % (R / 2));
            old[k] = (unsigned)(R / 2 + rng() % (R / 2));
            slots[k] = (unsigned)(rng() % 4000000);
        }
        CK(cudaMemcpy(d_rows, rows.data(), M * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_old, old.data(), M * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_slots, slots.data(), M * 4, cudaMemcpyHostToDevice));
        for (int grid : {37, 74, 148, 296}) {
            float t0 = timeit([&] { exchange<0, 4><<<grid, 256>>>((float4 *)h, dev, d_rows, d_old, d_slots, M, D4); });
            float t1 = timeit([&] { exchange<1, 4><<<grid, 256>>>((float4 *)h, dev, d_rows, d_old, d_slots, M, D4); });
            float t2 = timeit([&] { exchange<2, 4><<<grid, 256>>>((float4 *)h, dev, d_rows, d_old, d_slots, M, D4); });
            float t3 = timeit([&] { exchange<3, 1><<<grid, 256>>>((float4 *)h, dev, d_rows, d_old, d_slots, M, D4); });
            float t4 = timeit([&] { exchange<2, 1><<<grid, 256>>>((float4 *)h, dev, d_rows, d_old, d_slots, M, D4); });
            printf("exchange M=%6d grid=%3d | v1-order %.1fus | loads-first %.1fus | wb-stores-first %.1fus | split-roles %.1fus | wb-first unr1 %.1fus\n",
                   M, grid, t0, t1, t2, t3, t4);
        }
    }
    // copy-engine reference: one contiguous H2D of M rows
    for (int M : Ms) {
        float t = timeit([&] { cudaMemcpyAsync(dev, h, (size_t)M * D * 4, cudaMemcpyHostToDevice); });
        printf("memcpy H2D contiguous M=%d: %.1fus (%.1f GB/s)\n", M, t, (double)M * D * 4 / t / 1e3);
    }
    return 0;
}
