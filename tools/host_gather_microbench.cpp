// host_gather_microbench.cpp — CPU random-row gather cost on the GPU box (not
// product code): 8.4 GB table, 1800 random 256-B rows, 4-KB pages vs
// transparent huge pages, 1..8 threads, with/without whole-chunk prefetch.
// Build: g++ -O2 -std=c++17 -pthread -o host_gather_mb host_gather_microbench.cpp
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t R = 33000000, RB = 256, bytes = R * RB;
    FILE *f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[256] = {0};
    if (f) { fgets(buf, sizeof buf, f); fclose(f); }
    printf("THP enabled: %s", buf);
    for (int huge = 0; huge < 2; huge++) {
        char *t = (char *)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (huge) madvise(t, bytes, MADV_HUGEPAGE);
        else madvise(t, bytes, MADV_NOHUGEPAGE);
        memset(t, 1, bytes);
        std::vector<char> stage(8000 * RB);
        std::mt19937_64 rng(1);
        for (int nt : {1, 2, 4, 8}) {
            for (int pf = 0; pf < 2; pf++) {
                double best = 1e9;
                for (int it = 0; it < 20; it++) {
                    const int M = 1800;
                    std::vector<size_t> rows(M);
                    for (auto &x : rows) x = rng() % R;
                    std::atomic<int> next{0};
                    auto work = [&] {
                        for (;;) {
                            int i0 = next.fetch_add(16);
                            if (i0 >= M) break;
                            int i1 = std::min(M, i0 + 16);
                            if (pf)
                                for (int i = i0; i < i1; i++)
                                    for (size_t o = 0; o < RB; o += 64) __builtin_prefetch(t + rows[i] * RB + o, 0, 2);
                            for (int i = i0; i < i1; i++) memcpy(&stage[i * RB], t + rows[i] * RB, RB);
                        }
                    };
                    double t0 = now_us();
                    std::vector<std::thread> th;
                    for (int k = 1; k < nt; k++) th.emplace_back(work);
                    work();
                    for (auto &x : th) x.join();
                    best = std::min(best, now_us() - t0);
                }
                printf("%s threads=%d prefetch=%d: 1800 rows in %.1f us (incl. %d thread spawns)\n",
                       huge ? "THP " : "4KiB", nt, pf, best, nt - 1);
            }
        }
        munmap(t, bytes);
    }
    return 0;
}
