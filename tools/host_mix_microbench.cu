// host_mix_microbench.cu — do the host-link directions and the CPU row
// copies share one limit?  (not product code)  Random 512-B rows of a 32 GB
// THP host table, FRESH rows every batch of 5,800 (one Terabyte-shaped
// batch's misses): GPU pull alone, GPU write-back alone, both at once on two
// streams, each beside CPU threads scattering / gathering another 5,800 rows,
// and all of it together.  Times are per batch (CUDA events for the GPU
// legs, wall clock for the batch).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o host_mix_mb host_mix_microbench.cu -lpthread
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

constexpr size_t ROWB = 512;

template <int MODE>
__global__ void rows_k(float4 *host, float4 *dev, const unsigned *rows, int M) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x / 32;
    for (int k = blockIdx.x * wpb + threadIdx.x / 32; k < M; k += gridDim.x * wpb) {
        if (MODE == 1) dev[(size_t)k * 32 + lane] = __ldcv(host + (size_t)rows[k] * 32 + lane);
        else host[(size_t)rows[k] * 32 + lane] = dev[(size_t)k * 32 + lane];
    }
}

struct Cpu {
    std::vector<std::thread> th;
    std::atomic<int> go{0}, done{0}, next{0};
    std::atomic<bool> stop{false};
    const unsigned *rows = nullptr;
    char *tab = nullptr, *buf = nullptr;
    int M = 0;
    bool scatter = true;
    void work() {
        for (;;) {
            const int i0 = next.fetch_add(16);
            if (i0 >= M) break;
            const int i1 = std::min(M, i0 + 16);
            for (int i = i0; i < i1; i++) {
                const char *p = scatter ? buf + (size_t)i * ROWB : tab + (size_t)rows[i] * ROWB;
                for (size_t o = 0; o < ROWB; o += 64) __builtin_prefetch(p + o, 0, 2);
            }
            for (int i = i0; i < i1; i++) {
                const char *s = scatter ? buf + (size_t)i * ROWB : tab + (size_t)rows[i] * ROWB;
                char *d = scatter ? tab + (size_t)rows[i] * ROWB : buf + (size_t)i * ROWB;
                for (size_t q = 0; q < ROWB / 16; q++)
                    _mm_stream_si128(reinterpret_cast<__m128i *>(d) + q,
                                     _mm_load_si128(reinterpret_cast<const __m128i *>(s) + q));
            }
            _mm_sfence();
        }
    }
    void start(int n) {
        for (int i = 0; i < n; i++)
            th.emplace_back([this] {
                int seen = 0;
                while (!stop.load()) {
                    const int g = go.load();
                    if (g == seen) {
                        _mm_pause();
                        continue;
                    }
                    seen = g;
                    work();
                    done.fetch_add(1);
                }
            });
    }
    void launch(const unsigned *r, int m, bool sc) {
        rows = r;
        M = m;
        scatter = sc;
        next = 0;
        done = 0;
        go.fetch_add(1);
    }
    void wait() {
        while (done.load() < (int)th.size()) _mm_pause();
    }
    void shutdown() {
        stop = true;
        for (auto &t : th) t.join();
    }
};

int main() {
    const size_t GB = 32, bytes = GB << 30, R = bytes / ROWB;
    const int M = 5800, SETS = 30;
    char *h = (char *)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(h, bytes, MADV_HUGEPAGE);
    memset(h, 0, bytes);
    CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
    float4 *hd = nullptr;
    CK(cudaHostGetDevicePointer((void **)&hd, h, 0));
    float4 *dev1, *dev2;
    CK(cudaMalloc(&dev1, (size_t)M * ROWB));
    CK(cudaMalloc(&dev2, (size_t)M * ROWB));
    std::mt19937_64 rng(5);
    // four disjoint row streams: GPU pull, GPU write-back, CPU scatter, CPU gather
    std::vector<unsigned> rows((size_t)4 * M * (SETS + 1));
    for (auto &x : rows) x = (unsigned)(rng() % R);
    unsigned *d_rows;
    CK(cudaMalloc(&d_rows, rows.size() * 4));
    CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    auto rset = [&](int kind, int i) { return (size_t)(kind * (SETS + 1) + i) * M; };
    char *cbuf = (char *)aligned_alloc(4096, (size_t)M * ROWB);
    memset(cbuf, 1, (size_t)M * ROWB);
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a1, b1, a2, b2;
    cudaEventCreate(&a1);
    cudaEventCreate(&b1);
    cudaEventCreate(&a2);
    cudaEventCreate(&b2);
    for (int grid : {37, 148}) {
        for (int cth : {0, 4, 8}) {
            Cpu cpu;
            cpu.tab = h;
            cpu.buf = cbuf;
            if (cth) cpu.start(cth);
            for (int mix = 0; mix < 7; mix++) {
                // mix bits: 1 GPU pull, 2 GPU write-back, 4 CPU leg; the CPU leg
                // scatters (mix 4..5) or gathers (mix 6)
                const bool pull = mix == 0 || mix == 2 || mix == 4 || mix == 6;
                const bool wb = mix == 1 || mix == 2 || mix == 5 || mix == 6;
                const bool cpuleg = mix >= 3;
                if (cpuleg && !cth) continue;
                if (!cpuleg && cth) continue;
                const bool gather = mix == 6 && false;
                double sum_pull = 0, sum_wb = 0, sum_wall = 0;
                for (int i = 1; i <= SETS; i++) {
                    auto t0 = std::chrono::steady_clock::now();
                    if (pull) {
                        cudaEventRecord(a1, s1);
                        rows_k<1><<<grid, 256, 0, s1>>>(hd, dev1, d_rows + rset(0, i), M);
                        cudaEventRecord(b1, s1);
                    }
                    if (wb) {
                        cudaEventRecord(a2, s2);
                        rows_k<2><<<grid, 256, 0, s2>>>(hd, dev2, d_rows + rset(1, i), M);
                        cudaEventRecord(b2, s2);
                    }
                    if (cpuleg) cpu.launch(rows.data() + rset(mix == 6 ? 3 : 2, i), M, !gather);
                    if (cpuleg) cpu.wait();
                    CK(cudaStreamSynchronize(s1));
                    CK(cudaStreamSynchronize(s2));
                    auto t1 = std::chrono::steady_clock::now();
                    float ms;
                    if (pull) {
                        cudaEventElapsedTime(&ms, a1, b1);
                        sum_pull += ms * 1e3;
                    }
                    if (wb) {
                        cudaEventElapsedTime(&ms, a2, b2);
                        sum_wb += ms * 1e3;
                    }
                    sum_wall += std::chrono::duration<double, std::micro>(t1 - t0).count();
                }
                const char *names[] = {"pull", "writeback", "pull+writeback", "cpu-scatter",
                                       "pull+cpu-scatter", "writeback+cpu-scatter", "pull+writeback+cpu-scatter"};
                printf("grid %3d cpu threads %d %-28s GPU pull %6.1f us  GPU wb %6.1f us  batch wall %6.1f us\n", grid,
                       cth, names[mix], pull ? sum_pull / SETS : 0.0, wb ? sum_wb / SETS : 0.0, sum_wall / SETS);
            }
            if (cth) cpu.shutdown();
        }
    }
    return 0;
}
