// k_xfer.cu — the GPU side of [Collect] / [Exchange] / [Insert] (PAPER.md
// P:688-704) and the end-of-run write-back.
//
// Direction by direction, on measurements of this platform
// (profiles/r01_interference_microbench.txt, r01_host_gather.txt):
//   host -> HBM  SM zero-copy reads from a BOUNDED grid (8 CTAs): reads are
//                the benign direction (~1.2-1.6x on concurrent HBM kernels
//                vs ~6x for full-rate writes), and the GPU gathers the rows
//                itself: no CPU copy (random host rows cost ~31 ns/row/core
//                in this VM) and no per-batch API calls for sizes.
//   HBM -> host  the same kernel writes the victims, contiguously, into a
//                pinned host staging slot (sequential pages: few address
//                translations), raises a pinned flag when the last CTA is
//                done, and the CPU threads of the transfer engine scatter them
//                into the host tables (runtime.cu): random host rows are
//                translated by the CPU MMU, not the IOMMU the pulls use.
//   k_pullfill (transfer stream): for every fill k (slot s, missed row x,
//   previous resident o) of Plan(b), staging index i = prefix + k:
//       wb_stage[i] <- Storage[s]     if o is valid (dirty victim, P:693-696;
//                                     pinned host staging, zero-copy store)
//       Storage[s]  <- host[t][x]     zero-copy PCIe read
//   the same lane reads the victim before overwriting the slot.
#include "sp_internal.cuh"

namespace sp {

// Completion of Transfer(b) for the scatter thread: every CTA's staging stores
// are made visible system-wide, then the last CTA to arrive raises the pinned
// flag (and resets the counter for the next use of this ring slot).
__device__ __forceinline__ void publish_staged(const XferArgs &A) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned k = atomicAdd(A.done_ctr, 1u);
        if (k == gridDim.x - 1) {
            *A.done_ctr = 0u;
            __threadfence_system();
            *(volatile unsigned long long *)A.staged = (unsigned long long)(A.b + 1);
        }
    }
}

// G lanes per row, VPL float4 per lane, XU rows in flight per lane group.
// Per fill k (slot s, missed row x, previous resident o), staging i = prefix + k:
//   wb_stage[i] <- Storage[s]        if o is valid (dirty victim -> pinned staging)
//   Storage[s]  <- host[t][x]        zero-copy PCIe read (bounded grid)
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_pullfill(XferArgs A) {
    if (*A.err != NO_ERR) return;
    constexpr int XU = 4;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ uint32_t s_pref[65];
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    float4 *wbs = reinterpret_cast<float4 *>(A.wb_stage);
    uint32_t base_t0 = 0;  // staging rows of the tables before t0
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.m, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        const uint32_t ngroups = gridDim.x * gpb;
        for (uint32_t base = (blockIdx.x * gpb + threadIdx.x / G) * XU; base < total; base += ngroups * XU) {
            uint32_t slot[XU];
            size_t idx[XU];
            bool wb[XU];
            const float4 *src[XU];
#pragma unroll
            for (int r = 0; r < XU; r++) {
                const uint32_t item = base + r;
                slot[r] = EMPTY;
                if (item < total) {
                    const int tl = find_table(s_pref, tcount, item);
                    const size_t kk = (size_t)(t0 + tl) * g.n + (item - s_pref[tl]);
                    idx[r] = (size_t)base_t0 + item;
                    slot[r] = A.bb.fill_slot[kk];
                    wb[r] = A.bb.evict_row[kk] != EMPTY;
                    src[r] = reinterpret_cast<const float4 *>(A.host[t0 + tl] + (size_t)A.bb.fill_row[kk] * g.D);
                }
            }
            float4 x[XU][VPL];
#pragma unroll
            for (int r = 0; r < XU; r++)  // PCIe reads in flight first
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) x[r][q] = __ldcv(src[r] + lane + q * G);
#pragma unroll
            for (int r = 0; r < XU; r++)  // victims staged while the reads fly
                if (slot[r] != EMPTY && wb[r])
#pragma unroll
                    for (int q = 0; q < VPL; q++)
                        wbs[idx[r] * D4 + lane + q * G] = st[(size_t)slot[r] * D4 + lane + q * G];
#pragma unroll
            for (int r = 0; r < XU; r++)
                if (slot[r] != EMPTY)
#pragma unroll
                    for (int q = 0; q < VPL; q++) st[(size_t)slot[r] * D4 + lane + q * G] = x[r][q];
        }
        base_t0 += total;
    }
    publish_staged(A);
}

__global__ void __launch_bounds__(256) k_pullfill_generic(XferArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    float4 *wbs = reinterpret_cast<float4 *>(A.wb_stage);
    const int wpb = blockDim.x / 32;
    size_t base = 0;
    for (int t = 0; t < g.T; t++) {
        const uint32_t m = A.bb.m[t];
        const float *h = A.host[t];
        for (uint32_t k = blockIdx.x * wpb + threadIdx.x / 32; k < m; k += gridDim.x * wpb) {
            const size_t kk = (size_t)t * g.n + k, i = base + k;
            const uint32_t s = A.bb.fill_slot[kk], x = A.bb.fill_row[kk];
            const bool wb = A.bb.evict_row[kk] != EMPTY;
            for (int c = lane; c < D4; c += 32) {
                const float4 in = __ldcv(reinterpret_cast<const float4 *>(h + (size_t)x * g.D) + c);
                if (wb) wbs[i * D4 + c] = st[(size_t)s * D4 + c];
                st[(size_t)s * D4 + c] = in;
            }
        }
        base += m;
    }
    publish_staged(A);
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

cudaError_t launch_pullfill(const XferArgs &a, int ctas, cudaStream_t s) {
    const int grid = ctas > 0 ? ctas : 8;
    static bool once = false;
    if (!once) {
        apply_carveout(k_pullfill<16, 1>);
        apply_carveout(k_pullfill<32, 1>);
        apply_carveout(k_pullfill<32, 2>);
        apply_carveout(k_pullfill<32, 4>);
        apply_carveout(k_pullfill_generic);
        once = true;
    }
    switch (a.g.D / 4) {
        case 1: k_pullfill<1, 1><<<grid, 256, 0, s>>>(a); break;
        case 2: k_pullfill<2, 1><<<grid, 256, 0, s>>>(a); break;
        case 4: k_pullfill<4, 1><<<grid, 256, 0, s>>>(a); break;
        case 8: k_pullfill<8, 1><<<grid, 256, 0, s>>>(a); break;
        case 16: k_pullfill<16, 1><<<grid, 256, 0, s>>>(a); break;
        case 32: k_pullfill<32, 1><<<grid, 256, 0, s>>>(a); break;
        case 64: k_pullfill<32, 2><<<grid, 256, 0, s>>>(a); break;
        case 128: k_pullfill<32, 4><<<grid, 256, 0, s>>>(a); break;
        case 256: k_pullfill<32, 8><<<grid, 256, 0, s>>>(a); break;
        default: k_pullfill_generic<<<grid, 256, 0, s>>>(a); break;
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
