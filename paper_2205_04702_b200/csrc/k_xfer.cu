// k_xfer.cu — [Collect] + [Exchange] + [Insert] for the
// B200 host link, split by direction, plus the end-of-run write-back.
//
// Measured on this platform (profiles/r01_interference_microbench.txt,
// r01_xfer_microbench*.txt): SM-issued PCIe *writes* at full link rate slow a
// concurrent HBM-bound kernel ~6x, and reads queue behind posted writes, while
// reads from a bounded grid (~16 CTAs, ~30 GB/s) cost ~1.6x and writes from
// 1-2 CTAs (~12-20 GB/s) are nearly free.  So:
//
//   k_pull (transfer stream, bounded grid, reads only):
//     for every fill (slot s, missed row x) planned at Plan(b):
//       stage[k] <- Storage[s]      copy the dirty victim to HBM
//       Storage[s] <- host[t][x]    pull the missed row (zero-copy read)
//     the same lane does both, so the victim is captured before the overwrite.
//   k_writeback (write-back stream, 1-2 CTAs, writes only):
//       host[t][old] <- stage[k]    mandatory write-back of every valid victim
//                                   (P:716-718), rate-limited in the background
//   Pull(b) waits for WriteBack(b-F-1): a row evicted at Plan(b') is not in
//   B(b'+1..b'+F), so the first pull that can read it again is Pull(b'+F+1)
//   (RAW-4).
//
// No staging in host memory and no CPU gather/scatter: the paper's CPU-side
// Collect/Insert work disappears, the copies are issued by SMs.
#include "sp_internal.cuh"

namespace sp {

namespace {
constexpr int XFER_UNROLL = 8;  // rows in flight per lane group
constexpr int XFER_THREADS = 256;
}  // namespace

// G lanes per row, VPL float4 per lane.
template <int G, int VPL>
__global__ void __launch_bounds__(XFER_THREADS) k_pull(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ uint32_t s_pref[65];
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    float4 *stage = reinterpret_cast<float4 *>(A.stage);
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.m, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        const uint32_t ngroups = gridDim.x * gpb;
        for (uint32_t base = (blockIdx.x * gpb + threadIdx.x / G) * XFER_UNROLL; base < total;
             base += ngroups * XFER_UNROLL) {
            uint32_t slot[XFER_UNROLL];
            size_t kk[XFER_UNROLL];
            bool wb[XFER_UNROLL];
            const float4 *src[XFER_UNROLL];
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++) {
                const uint32_t item = base + r;
                slot[r] = EMPTY;
                if (item < total) {
                    const int tl = find_table(s_pref, tcount, item);
                    const int t = t0 + tl;
                    kk[r] = (size_t)t * g.n + (item - s_pref[tl]);
                    slot[r] = A.bb.fill_slot[kk[r]];
                    wb[r] = A.bb.evict_row[kk[r]] != EMPTY;
                    src[r] = reinterpret_cast<const float4 *>(A.host[t] + (size_t)A.bb.fill_row[kk[r]] * g.D);
                }
            }
            // PCIe reads in flight first (nothing ahead of them on the link) ...
            float4 x[XFER_UNROLL][VPL];
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) x[r][q] = __ldcv(src[r] + lane + q * G);
            // ... meanwhile the victims move HBM -> HBM staging ...
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY && wb[r])
#pragma unroll
                    for (int q = 0; q < VPL; q++)
                        stage[kk[r] * D4 + lane + q * G] = st[(size_t)slot[r] * D4 + lane + q * G];
            // ... then the fills overwrite the freed slots
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) st[(size_t)slot[r] * D4 + lane + q * G] = x[r][q];
        }
    }
}

__global__ void __launch_bounds__(256) k_pull_generic(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    float4 *stage = reinterpret_cast<float4 *>(A.stage);
    const int wpb = blockDim.x / 32;
    for (int t = 0; t < g.T; t++) {
        const uint32_t m = A.bb.m[t];
        const float *h = A.host[t];
        for (uint32_t k = blockIdx.x * wpb + threadIdx.x / 32; k < m; k += gridDim.x * wpb) {
            const size_t kk = (size_t)t * g.n + k;
            const uint32_t s = A.bb.fill_slot[kk], x = A.bb.fill_row[kk], o = A.bb.evict_row[kk];
            for (int c = lane; c < D4; c += 32) {
                const float4 in = __ldcv(reinterpret_cast<const float4 *>(h + (size_t)x * g.D) + c);
                if (o != EMPTY) stage[kk * D4 + c] = st[(size_t)s * D4 + c];
                st[(size_t)s * D4 + c] = in;
            }
        }
    }
}

// write-back of the staged victims of one batch (PCIe writes only).  Few
// CTAs bound the write rate (a full-rate write stream slows concurrent HBM
// kernels ~6x); WB_UNROLL rows in flight per lane group hide the index/stage
// load latency so those few CTAs still reach ~15-25 GB/s.
template <int G, int VPL>
__global__ void __launch_bounds__(XFER_THREADS) k_writeback(XferArgs A) {
    if (*A.err != NO_ERR) return;
    constexpr int WB_UNROLL = 8;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ uint32_t s_pref[65];
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    const float4 *stage = reinterpret_cast<const float4 *>(A.stage);
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.m, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        const uint32_t ngroups = gridDim.x * gpb;
        for (uint32_t base = (blockIdx.x * gpb + threadIdx.x / G) * WB_UNROLL; base < total;
             base += ngroups * WB_UNROLL) {
            size_t kk[WB_UNROLL];
            uint32_t old[WB_UNROLL];
            float *h[WB_UNROLL];
#pragma unroll
            for (int r = 0; r < WB_UNROLL; r++) {
                const uint32_t item = base + r;
                old[r] = EMPTY;
                if (item < total) {
                    const int tl = find_table(s_pref, tcount, item);
                    const int t = t0 + tl;
                    kk[r] = (size_t)t * g.n + (item - s_pref[tl]);
                    old[r] = A.bb.evict_row[kk[r]];
                    h[r] = A.host[t];
                }
            }
            float4 v[WB_UNROLL][VPL];
#pragma unroll
            for (int r = 0; r < WB_UNROLL; r++)
                if (old[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) v[r][q] = stage[kk[r] * D4 + lane + q * G];
#pragma unroll
            for (int r = 0; r < WB_UNROLL; r++)
                if (old[r] != EMPTY) {
                    float4 *dst = reinterpret_cast<float4 *>(h[r] + (size_t)old[r] * g.D) + lane;
#pragma unroll
                    for (int q = 0; q < VPL; q++) dst[q * G] = v[r][q];
                }
        }
    }
}

__global__ void __launch_bounds__(256) k_writeback_generic(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    const float4 *stage = reinterpret_cast<const float4 *>(A.stage);
    const int wpb = blockDim.x / 32;
    for (int t = 0; t < g.T; t++) {
        const uint32_t m = A.bb.m[t];
        float *h = A.host[t];
        for (uint32_t k = blockIdx.x * wpb + threadIdx.x / 32; k < m; k += gridDim.x * wpb) {
            const size_t kk = (size_t)t * g.n + k;
            const uint32_t o = A.bb.evict_row[kk];
            if (o == EMPTY) continue;
            for (int c = lane; c < D4; c += 32) reinterpret_cast<float4 *>(h + (size_t)o * g.D)[c] = stage[kk * D4 + c];
        }
    }
}

// write back every resident slot (sp_flush)
__global__ void __launch_bounds__(256) k_flush(FlushArgs A) {
    const int D4 = A.g.D / 4;
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x / 32;
    for (long long s = (long long)blockIdx.x * wpb + threadIdx.x / 32; s < A.S_total;
         s += (long long)gridDim.x * wpb) {
        const uint32_t id = A.resident[s];
        if (id == EMPTY) continue;
        int t = 0;
        while ((long long)A.slot_base[t + 1] <= s) t++;
        float4 *dst = reinterpret_cast<float4 *>(A.host[t] + (size_t)id * A.g.D);
        const float4 *src = reinterpret_cast<const float4 *>(A.storage) + (size_t)s * D4;
        for (int c = lane; c < D4; c += 32) dst[c] = src[c];
    }
}

static int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

#define SP_DISPATCH_XFER(KERNEL, GRID, ARGS, STREAM)                                  \
    switch ((ARGS).g.D / 4) {                                                          \
        case 1: KERNEL<1, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;          \
        case 2: KERNEL<2, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;          \
        case 4: KERNEL<4, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;          \
        case 8: KERNEL<8, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;          \
        case 16: KERNEL<16, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;        \
        case 32: KERNEL<32, 1><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;        \
        case 64: KERNEL<32, 2><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;        \
        case 128: KERNEL<32, 4><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;       \
        case 256: KERNEL<32, 8><<<GRID, XFER_THREADS, 0, STREAM>>>(ARGS); break;       \
        default: KERNEL##_generic<<<GRID, 256, 0, STREAM>>>(ARGS); break;              \
    }

cudaError_t launch_pull(const XferArgs &a, int ctas, cudaStream_t s) {
    const int grid = ctas > 0 ? ctas : 16;
    SP_DISPATCH_XFER(k_pull, grid, a, s);
    return cudaGetLastError();
}

cudaError_t launch_writeback(const XferArgs &a, int ctas, cudaStream_t s) {
    const int grid = ctas > 0 ? ctas : 2;
    SP_DISPATCH_XFER(k_writeback, grid, a, s);
    return cudaGetLastError();
}

cudaError_t launch_flush(const FlushArgs &a, cudaStream_t s) {
    long long blocks = ((long long)a.S_total + 7) / 8;
    long long cap = (long long)sm_count() * 8;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    k_flush<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sp
