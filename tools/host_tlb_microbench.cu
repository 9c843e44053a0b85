// host_tlb_microbench.cu — cost of GPU address translation for random rows of
// a large pinned host table (not product code).  Each launch moves a FRESH
// set of M random 256-B rows (cold translations), unlike a loop over the same
// rows.  Host table allocated three ways: cudaHostAlloc, mmap + THP +
// cudaHostRegister, mmap (4 KB pages) + cudaHostRegister.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o host_tlb_mb host_tlb_microbench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
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

// plain pull: 16 lanes x float4 per row; MODE 1 pull, 2 write-back
template <int MODE>
__global__ void plain(float4 *host, float4 *dev, const unsigned *rows, const unsigned *slots, int M) {
    const int G = 16, gpb = blockDim.x / G, lane = threadIdx.x % G;
    for (int k = blockIdx.x * gpb + threadIdx.x / G; k < M; k += gridDim.x * gpb) {
        if (MODE == 1) dev[(size_t)slots[k] * 16 + lane] = __ldcv(host + (size_t)rows[k] * 16 + lane);
        else host[(size_t)rows[k] * 16 + lane] = dev[(size_t)slots[k] * 16 + lane];
    }
}

int main() {
    const size_t R = 33000000, S = 3400000, rowb = 256;
    const size_t bytes = R * rowb;
    const int M = 1800, SETS = 60;
    float4 *dev;
    CK(cudaMalloc(&dev, S * rowb));
    std::mt19937_64 rng(7);
    std::vector<unsigned> rows((size_t)M * SETS), slots((size_t)M * SETS);
    for (auto &x : rows) x = rng() % R;
    for (auto &x : slots) x = rng() % S;
    unsigned *d_rows, *d_slots;
    CK(cudaMalloc(&d_rows, rows.size() * 4));
    CK(cudaMalloc(&d_slots, slots.size() * 4));
    CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_slots, slots.data(), slots.size() * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int kind = 3; kind >= 0; kind--) {
        void *h = nullptr;
        const char *name = kind == 0 ? "cudaHostAlloc" : kind == 1 ? "mmap+THP+register" : kind == 2 ? "mmap-4K+register" : "cuMemCreate(HOST_NUMA)";
        CUmemGenericAllocationHandle vh = 0;
        size_t vbytes = 0;
        if (kind == 3) {
            CUmemAllocationProp prop = {};
            prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
            prop.location.id = 0;
            size_t gmin = 0, grec = 0;
            cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
            cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
            vbytes = (bytes + grec - 1) / grec * grec;
            CUresult r = cuMemCreate(&vh, vbytes, &prop, 0);
            CUdeviceptr va = 0;
            if (r == CUDA_SUCCESS) r = cuMemAddressReserve(&va, vbytes, grec, 0, 0);
            if (r == CUDA_SUCCESS) r = cuMemMap(va, vbytes, 0, vh, 0);
            CUmemAccessDesc acc[2] = {};
            acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            acc[0].location.id = 0;
            acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
            acc[1].location.id = 0;
            acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            if (r == CUDA_SUCCESS) r = cuMemSetAccess(va, vbytes, acc, 2);
            printf("cuMemCreate HOST_NUMA: granularity min %zu rec %zu -> %d\n", gmin, grec, (int)r);
            if (r != CUDA_SUCCESS) continue;
            h = (void *)va;
            memset(h, 0, bytes);  // CPU access through the same VA
            ((float *)h)[12345] = 1.f;
        } else if (kind == 0) {
            CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
        } else {
            h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
            madvise(h, bytes, kind == 1 ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
            memset(h, 0, bytes);
            CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
        }
        float4 *hd = (float4 *)h;
        if (kind != 3) CK(cudaHostGetDevicePointer((void **)&hd, h, 0));
        for (int mode = 1; mode <= 2; mode++)
            for (int grid : {8, 16, 37}) {
                // warm-up launch on set 0 (same rows: warm translations)
                for (int i = 0; i < 3; i++) (mode == 1 ? plain<1> : plain<2>)<<<grid, 256>>>(hd, dev, d_rows, d_slots, M);
                cudaEventRecord(a);
                for (int i = 0; i < 20; i++) (mode == 1 ? plain<1> : plain<2>)<<<grid, 256>>>(hd, dev, d_rows, d_slots, M);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float warm;
                cudaEventElapsedTime(&warm, a, b);
                cudaEventRecord(a);
                for (int i = 1; i < SETS; i++)
                    (mode == 1 ? plain<1> : plain<2>)<<<grid, 256>>>(hd, dev, d_rows + (size_t)i * M, d_slots + (size_t)i * M, M);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float cold;
                cudaEventElapsedTime(&cold, a, b);
                printf("%-18s %-9s grid %3d: same rows %6.1f us/launch | fresh rows %6.1f us/launch\n", name,
                       mode == 1 ? "pull" : "writeback", grid, warm * 1000 / 20, cold * 1000 / (SETS - 1));
            }
        if (kind == 3) {
            cuMemUnmap((CUdeviceptr)h, vbytes);
            cuMemAddressFree((CUdeviceptr)h, vbytes);
            cuMemRelease(vh);
        } else if (kind == 0) cudaFreeHost(h);
        else {
            cudaHostUnregister(h);
            munmap(h, bytes);
        }
    }
    return 0;
}
