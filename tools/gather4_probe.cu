// gather4_probe.cu — does TMA tile::gather4 fetch 4 arbitrary rows of a 2-D
// fp32 matrix [R][D] into shared memory, and with which box?  (not product
// code; settles the tensor-map convention before k_bwd_tile uses it)
// Also times per-row bulk copies vs gather4 for 106,496 random 512-B rows.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

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

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, const int *rows, float *out, int D) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(4 * D * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5, %6}], [%7];" ::"r"(sa(sm)),
            "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(sa(&bar))
            : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok)
                         : "r"(sa(&bar))
                         : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * D; i += blockDim.x) out[i] = sm[i];
}

// timing: each warp takes groups of 4 rows (gather4) or 1 row per lane (bulk), TR rows per round
template <bool G4>
__global__ void __launch_bounds__(32) rate(const __grid_constant__ CUtensorMap tm, const float *mat, const int *rows,
                                           int M, int D, float *sink) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int TR = 16;
    uint32_t par = 0;
    float acc = 0.f;
    for (int base = blockIdx.x * TR; base < M; base += gridDim.x * TR) {
        const int n = min(TR, M - base);
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * D * 4) : "memory");
        __syncwarp();
        if (G4) {
            if (lane < n / 4)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3, %4, %5, %6}], [%7];" ::"r"(sa(sm + lane * 4 * D)),
                    "l"(&tm), "r"(0), "r"(rows[base + 4 * lane]), "r"(rows[base + 4 * lane + 1]), "r"(rows[base + 4 * lane + 2]),
                    "r"(rows[base + 4 * lane + 3]), "r"(sa(&bar))
                    : "memory");
        } else {
            if (lane < n)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 sa(sm + lane * D)),
                             "l"(mat + (size_t)rows[base + lane] * D), "r"(D * 4), "r"(sa(&bar))
                             : "memory");
        }
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok)
                         : "r"(sa(&bar)), "r"(par)
                         : "memory");
        par ^= 1;
        acc += sm[lane];
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (acc == 12345.f) sink[0] = acc;
}

typedef CUresult (*encode_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 4 << 20, D = 128, M = 106496;
    float *mat;
    CK(cudaMalloc(&mat, (size_t)R * D * 4));
    std::vector<float> h((size_t)1024 * D);
    for (size_t i = 0; i < h.size(); i++) h[i] = (float)i;
    CK(cudaMemcpy(mat, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    encode_t enc = (encode_t)fn;
    int rows_h[4] = {5, 17, 3, 1000};
    int *rows_d;
    CK(cudaMalloc(&rows_d, sizeof(int) * M));
    CK(cudaMemcpy(rows_d, rows_h, sizeof rows_h, cudaMemcpyHostToDevice));
    float *out;
    CK(cudaMalloc(&out, 4 * D * 4));
    for (int boxr : {1}) {  // (box rows 4: illegal instruction -- gather4 takes a one-row box)
        CUtensorMap tm;
        cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)R}, gstr[1] = {(cuuint64_t)D * 4};
        cuuint32_t box[2] = {(cuuint32_t)D, (cuuint32_t)boxr}, es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, mat, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box {%d, %d}: encode -> %d\n", D, boxr, (int)r);
        if (r) continue;
        CK(cudaMemset(out, 0, 4 * D * 4));
        probe<<<1, 128, 4 * D * 4>>>(tm, rows_d, out, D);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  launch -> %s\n", cudaGetErrorString(e));
        if (e) return 1;
        std::vector<float> o(4 * D);
        CK(cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int k = 0; k < 4; k++)
            for (int c = 0; c < D; c++)
                if (o[k * D + c] != (float)(rows_h[k] * D + c) && rows_h[k] < 1024) bad++;
        printf("  rows 5,17,3: mismatches %d (o[0]=%g want %g; o[D]=%g want %g)\n", bad, o[0], 5.f * D, o[D], 17.f * D);
    }
    // rate: random rows
    std::mt19937 rng(3);
    std::vector<int> rr(M);
    for (auto &x : rr) x = (int)(rng() % R);
    CK(cudaMemcpy(rows_d, rr.data(), sizeof(int) * M, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)R}, gstr[1] = {(cuuint64_t)D * 4};
    cuuint32_t box[2] = {(cuuint32_t)D, 1}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, mat, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int g4 = 0; g4 < 2; g4++)
        for (int grid : {148 * 6, 148 * 13}) {
            for (int it = 0; it < 2; it++) {
                cudaEventRecord(a);
                if (g4) rate<true><<<grid, 32, 16 * D * 4>>>(tm, mat, rows_d, M, D, out);
                else rate<false><<<grid, 32, 16 * D * 4>>>(tm, mat, rows_d, M, D, out);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (it) printf("%s grid %d: %d rows of %d B in %.1f us = %.0f GB/s\n", g4 ? "gather4" : "bulk/row", grid, M,
                               D * 4, ms * 1e3, (double)M * D * 4 / (ms * 1e-3) / 1e9);
            }
        }
    return 0;
}
