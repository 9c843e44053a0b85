// k_xfer.cu — [Collect] + [Exchange] + [Insert] fused into one zero-copy
// kernel, and the end-of-run write-back.
//
// For every fill (slot s, missed row x) planned at Plan(b), with the slot's
// previous resident row o (a valid victim):
//   host[t][o] <- Storage[s]   write-back of the dirty victim (mandatory:
//                              every cached row was trained, P:693-696,
//                              P:716-718), then
//   Storage[s] <- host[t][x]   pull of the missed row into the freed slot.
// The same lane does both for a slot, so the read of the victim precedes the
// write of the new row.  The host tables are pinned + mapped: SMs issue the
// PCIe reads/writes directly (16-byte vectors, several rows in flight per
// lane group), so there are no staging buffers and no CPU gather/scatter —
// the paper's CPU-side Collect/Insert work disappears.  Runs on its own
// stream with a bounded grid so it overlaps the HBM-bound Train kernels
// (the paper's "Collect overlapped with Train").
#include "sp_internal.cuh"

namespace sp {

namespace {
constexpr int XFER_UNROLL = 4;  // rows in flight per lane group
}  // namespace

// G lanes per row, VPL float4 per lane.
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_xfer(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ uint32_t s_pref[65];
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (int k = 0; k < tcount; k++) { s_pref[k] = run; run += A.bb.m[t0 + k]; }
            s_pref[tcount] = run;
        }
        __syncthreads();
        const uint32_t total = s_pref[tcount];
        const uint32_t ngroups = gridDim.x * gpb;
        for (uint32_t base = (blockIdx.x * gpb + threadIdx.x / G) * XFER_UNROLL; base < total;
             base += ngroups * XFER_UNROLL) {
            uint32_t slot[XFER_UNROLL], row[XFER_UNROLL], old[XFER_UNROLL];
            const float4 *src[XFER_UNROLL];
            float4 *wb[XFER_UNROLL];
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++) {
                const uint32_t item = base + r;
                slot[r] = EMPTY;
                if (item < total) {
                    int tl = 0;
                    while (s_pref[tl + 1] <= item) tl++;
                    const int t = t0 + tl;
                    const size_t k = (size_t)t * g.n + (item - s_pref[tl]);
                    slot[r] = A.bb.fill_slot[k];
                    row[r] = A.bb.fill_row[k];
                    old[r] = A.bb.evict_row[k];
                    float *h = A.host[t];
                    src[r] = reinterpret_cast<const float4 *>(h + (size_t)row[r] * g.D);
                    wb[r] = old[r] != EMPTY ? reinterpret_cast<float4 *>(h + (size_t)old[r] * g.D) : nullptr;
                }
            }
            // write-back of valid victims (Storage -> host)
            float4 v[XFER_UNROLL][VPL];
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY && wb[r])
#pragma unroll
                    for (int q = 0; q < VPL; q++) v[r][q] = st[(size_t)slot[r] * D4 + lane + q * G];
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY && wb[r])
#pragma unroll
                    for (int q = 0; q < VPL; q++) wb[r][lane + q * G] = v[r][q];
            // pull of missed rows (host -> Storage): all loads first
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) v[r][q] = __ldcv(src[r] + lane + q * G);
#pragma unroll
            for (int r = 0; r < XFER_UNROLL; r++)
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) st[(size_t)slot[r] * D4 + lane + q * G] = v[r][q];
        }
    }
}

__global__ void __launch_bounds__(256) k_xfer_generic(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    const int wpb = blockDim.x / 32;
    for (int t = 0; t < g.T; t++) {
        const uint32_t m = A.bb.m[t];
        float *h = A.host[t];
        for (uint32_t k = blockIdx.x * wpb + threadIdx.x / 32; k < m; k += gridDim.x * wpb) {
            const size_t kk = (size_t)t * g.n + k;
            const uint32_t s = A.bb.fill_slot[kk], x = A.bb.fill_row[kk], o = A.bb.evict_row[kk];
            for (int c = lane; c < D4; c += 32) {
                if (o != EMPTY)
                    reinterpret_cast<float4 *>(h + (size_t)o * g.D)[c] = st[(size_t)s * D4 + c];
                st[(size_t)s * D4 + c] = __ldcv(reinterpret_cast<const float4 *>(h + (size_t)x * g.D) + c);
            }
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

cudaError_t launch_transfer(const XferArgs &a, int max_ctas, cudaStream_t s) {
    const int D4 = a.g.D / 4;
    const int G = D4 >= 32 ? 32 : D4;
    const long long upper = (long long)a.g.T * a.g.n;  // fills <= uniques <= n per table
    long long blocks = (upper + (256 / G) * XFER_UNROLL - 1) / ((256 / G) * XFER_UNROLL);
    int grid = (int)(blocks < max_ctas ? blocks : max_ctas);
    if (grid < 1) grid = 1;
    switch (D4) {
        case 1: k_xfer<1, 1><<<grid, 256, 0, s>>>(a); break;
        case 2: k_xfer<2, 1><<<grid, 256, 0, s>>>(a); break;
        case 4: k_xfer<4, 1><<<grid, 256, 0, s>>>(a); break;
        case 8: k_xfer<8, 1><<<grid, 256, 0, s>>>(a); break;
        case 16: k_xfer<16, 1><<<grid, 256, 0, s>>>(a); break;
        case 32: k_xfer<32, 1><<<grid, 256, 0, s>>>(a); break;
        case 64: k_xfer<32, 2><<<grid, 256, 0, s>>>(a); break;
        case 128: k_xfer<32, 4><<<grid, 256, 0, s>>>(a); break;
        case 256: k_xfer<32, 8><<<grid, 256, 0, s>>>(a); break;
        default: k_xfer_generic<<<grid, 256, 0, s>>>(a); break;
    }
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
