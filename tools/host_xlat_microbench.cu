// host_xlat_microbench.cu — random 512-B rows of a large host table, per page
// size of the host allocation (not product code).  The scratchpad's transfer
// moves ~5.8k random rows each way per Terabyte-shaped batch; this measures
// what that costs on the GPU side (zero-copy pulls / write-backs from SMs, by
// grid size) and on the CPU side (row-copy threads), for FRESH rows every
// launch, with the host table on 4 KB / THP (2 MB) / hugetlb 2 MB / hugetlb
// 1 GB pages.  hugetlb pages are reserved through /proc/sys/vm (root on the
// GPU box) and released at the end.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o host_xlat_mb host_xlat_microbench.cu -lpthread
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#ifndef MAP_HUGE_1GB
#define MAP_HUGE_1GB (30 << 26)
#endif
#ifndef MAP_HUGE_2MB
#define MAP_HUGE_2MB (21 << 26)
#endif

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

constexpr size_t ROWB = 512;  // D = 128 fp32

// one warp per row (32 lanes x 16 B); MODE 1 pull host->dev, 2 write-back dev->host
template <int MODE>
__global__ void rows_k(float4 *host, float4 *dev, const unsigned *rows, int M) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x / 32;
    for (int k = blockIdx.x * wpb + threadIdx.x / 32; k < M; k += gridDim.x * wpb) {
        if (MODE == 1) dev[(size_t)k * 32 + lane] = __ldcv(host + (size_t)rows[k] * 32 + lane);
        else host[(size_t)rows[k] * 32 + lane] = dev[(size_t)k * 32 + lane];
    }
}

static void write_file(const char *p, const std::string &v) {
    FILE *f = fopen(p, "w");
    if (!f) return;
    fputs(v.c_str(), f);
    fclose(f);
}

static long read_long(const char *p) {
    FILE *f = fopen(p, "r");
    if (!f) return -1;
    long v = -1;
    if (fscanf(f, "%ld", &v) != 1) v = -1;
    fclose(f);
    return v;
}

// CPU gather of M random rows into a contiguous buffer with `nth` threads
// (chunks of 16 rows: every line of the chunk prefetched, then copied)
static double cpu_gather_us(const char *tab, char *out, const unsigned *rows, int M, int nth, bool scatter) {
    std::atomic<int> next{0};
    auto work = [&] {
        for (;;) {
            const int i0 = next.fetch_add(16);
            if (i0 >= M) break;
            const int i1 = std::min(M, i0 + 16);
            for (int i = i0; i < i1; i++) {
                const char *p = scatter ? out + (size_t)i * ROWB : tab + (size_t)rows[i] * ROWB;
                for (size_t o = 0; o < ROWB; o += 64) __builtin_prefetch(p + o, 0, 2);
                if (scatter) {
                    const char *q = tab + (size_t)rows[i] * ROWB;
                    __builtin_prefetch(q, 1, 2);
                }
            }
            for (int i = i0; i < i1; i++) {
                const char *s = scatter ? out + (size_t)i * ROWB : tab + (size_t)rows[i] * ROWB;
                char *d = scatter ? const_cast<char *>(tab) + (size_t)rows[i] * ROWB : out + (size_t)i * ROWB;
                for (size_t q = 0; q < ROWB / 16; q++)
                    _mm_stream_si128(reinterpret_cast<__m128i *>(d) + q,
                                     _mm_load_si128(reinterpret_cast<const __m128i *>(s) + q));
            }
            _mm_sfence();
        }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int k = 1; k < nth; k++) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count();
}

int main(int argc, char **argv) {
    const size_t GB = argc > 1 ? atol(argv[1]) : 32;  // table size
    const size_t bytes = GB << 30;
    const size_t R = bytes / ROWB;
    const int M = 5800, SETS = 40;
    printf("table %zu GB, %zu rows of %zu B, %d fresh random rows per launch, %d launches\n", GB, R, ROWB, M, SETS);
    float4 *dev;
    CK(cudaMalloc(&dev, (size_t)M * ROWB));
    std::mt19937_64 rng(11);
    std::vector<unsigned> rows((size_t)M * (SETS + 1));
    for (auto &x : rows) x = (unsigned)(rng() % R);
    unsigned *d_rows;
    CK(cudaMalloc(&d_rows, rows.size() * 4));
    CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    char *cbuf = (char *)aligned_alloc(4096, (size_t)M * ROWB);
    memset(cbuf, 1, (size_t)M * ROWB);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const long nr1g0 = read_long("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages");
    const long nr2m0 = read_long("/sys/kernel/mm/hugepages/hugepages-2048kB/nr_hugepages");
    FILE *thp = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char thpbuf[128] = {};
    if (thp) {
        if (!fgets(thpbuf, sizeof thpbuf, thp)) thpbuf[0] = 0;
        fclose(thp);
    }
    printf("THP enabled: %s", thpbuf);
    for (int kind = 0; kind < 4; kind++) {
        const char *name = kind == 0 ? "mmap-4K" : kind == 1 ? "mmap+THP" : kind == 2 ? "hugetlb-2M" : "hugetlb-1G";
        void *h = MAP_FAILED;
        if (kind <= 1) {
            h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
            if (h != MAP_FAILED) madvise(h, bytes, kind == 1 ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
        } else if (kind == 2) {
            write_file("/sys/kernel/mm/hugepages/hugepages-2048kB/nr_hugepages", std::to_string(bytes >> 21));
            printf("hugetlb 2M pages reserved: %ld (wanted %zu)\n",
                   read_long("/sys/kernel/mm/hugepages/hugepages-2048kB/nr_hugepages"), bytes >> 21);
            h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB | MAP_HUGE_2MB,
                     -1, 0);
        } else {
            write_file("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages", std::to_string(GB));
            printf("hugetlb 1G pages reserved: %ld (wanted %zu)\n",
                   read_long("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages"), GB);
            h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB | MAP_HUGE_1GB,
                     -1, 0);
        }
        if (h == MAP_FAILED) {
            printf("%-11s mmap failed: %s\n", name, strerror(errno));
            continue;
        }
        auto t0 = std::chrono::steady_clock::now();
        memset(h, 0, bytes);
        auto t1 = std::chrono::steady_clock::now();
        printf("%-11s first touch %.1f s\n", name, std::chrono::duration<double>(t1 - t0).count());
        CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
        float4 *hd = nullptr;
        CK(cudaHostGetDevicePointer((void **)&hd, h, 0));
        for (int mode = 1; mode <= 2; mode++)
            for (int grid : {16, 37, 74, 148, 296}) {
                for (int threads : {128, 256}) {
                    (mode == 1 ? rows_k<1> : rows_k<2>)<<<grid, threads>>>(hd, dev, d_rows, M);
                    CK(cudaDeviceSynchronize());
                    cudaEventRecord(a);
                    for (int i = 1; i <= SETS; i++)
                        (mode == 1 ? rows_k<1> : rows_k<2>)<<<grid, threads>>>(hd, dev, d_rows + (size_t)i * M, M);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    const double us = ms * 1000 / SETS;
                    printf("%-11s GPU %-9s grid %3d x %3d: %7.1f us/launch  %5.1f ns/row  %5.1f GB/s\n", name,
                           mode == 1 ? "pull" : "writeback", grid, threads, us, us * 1e3 / M,
                           (double)M * ROWB / us / 1e3);
                }
            }
        for (int scatter = 0; scatter <= 1; scatter++)
            for (int nth : {1, 2, 4, 8, 12}) {
                double tot = 0;
                for (int i = 1; i <= 10; i++)
                    tot += cpu_gather_us((const char *)h, cbuf, rows.data() + (size_t)i * M, M, nth, scatter);
                const double us = tot / 10;
                printf("%-11s CPU %-9s threads %2d: %7.1f us/batch  %5.1f ns/row\n", name,
                       scatter ? "scatter" : "gather", nth, us, us * 1e3 / M);
            }
        CK(cudaHostUnregister(h));
        munmap(h, bytes);
    }
    if (nr2m0 >= 0) write_file("/sys/kernel/mm/hugepages/hugepages-2048kB/nr_hugepages", std::to_string(nr2m0));
    if (nr1g0 >= 0) write_file("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages", std::to_string(nr1g0));
    return 0;
}
