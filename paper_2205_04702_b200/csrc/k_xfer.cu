// k_xfer.cu — [Collect] + [Exchange] + [Insert] as ONE
// GPU kernel per batch, and the end-of-run write-back (sp_flush).
//
// The paper moves rows with CPU threads and PCIe DMA.
// Here the GPU moves both directions itself, with TMA bulk copies
// (cp.async.bulk) between HBM, shared memory and the caller's pinned host
// tables (mapped, UVA):
//
//   for every fill k of Plan(b) (slot s, missed row x, previous resident o):
//     victim   Storage[s]  --bulk-->  smem  --bulk-->  host[t][o]   (if o valid:
//              the dirty write-back of P:693-696 / P:716-718, RAW-4 P:759-761)
//     fill     host[t][x]  --bulk-->  smem  --bulk-->  Storage[s]
//   both loads of an item land in shared memory before either store is
//   issued, so the victim is read before its slot is overwritten.
//
// Why this shape (profiles/r01_tma_xfer_microbench*.txt, measured on B200):
// - host-link throughput from SM-issued traffic grows ~3.5 GB/s per SM and
//   saturates near 30-40 GB/s, whatever the per-CTA queue depth, so the grid
//   is a small number of one-warp CTAs (`ctas`, default 16);
// - 16-B zero-copy stores from a few CTAs slowed a concurrent HBM gather up to
//   ~4x, TMA bulk stores of whole rows ~1.1-1.5x;
// - no CPU thread touches a row: no host gather/scatter, no staging, no
//   per-batch host API call.
//
// Ordering.  Items of one launch touch distinct slots and distinct host rows
// (a slot is a victim at most once per Plan; old residents and missed IDs are
// disjoint).  Transfers run in batch order on one stream and each launch
// waits for its bulk stores to complete before exiting, so a row written back
// at Transfer(b) is in host memory before any later Transfer pulls it again
// (RAW-4).
#include "sp_internal.cuh"

namespace sp {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "SP_MBW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra SP_MBW;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global (HBM or mapped host) -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// shared -> global (HBM or mapped host), bulk async-group of the issuing thread
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace

// One warp per CTA.  The flattened fill list of all tables (table_prefix over
// m[t]) is split into contiguous shares, one per CTA; a share is moved in
// rounds of nb items (one per lane) through XS shared-memory stages, so the
// loads of the next XS-1 rounds are in flight while a round is stored.
constexpr int XS = 4;

__global__ void __launch_bounds__(32) k_exchange(XferArgs A, int nb) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[XS];
    __shared__ uint32_t s_pref[65];
    __shared__ float *s_dst_host[XS][32];   // write-back destination (nullptr: vacant slot)
    __shared__ uint32_t s_slot[XS][32];
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const uint32_t rowb = (uint32_t)g.D * 4u;
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < XS; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase_ctr = 0;  // rounds completed on each stage so far (parity source)
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        // table_prefix uses 32 threads and __syncthreads (one warp: fine)
        table_prefix(A.bb.m, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
        const uint32_t lo = min(total, blockIdx.x * per), hi = min(total, lo + per);
        const uint32_t nround = hi > lo ? (hi - lo + nb - 1) / nb : 0;
        auto vbuf = [&](int s, int i) { return sm + ((size_t)s * nb + i) * 2 * rowb; };
        auto issue = [&](uint32_t r) {
            const int s = (int)((phase_ctr + r) % XS);
            const uint32_t k0 = lo + r * nb;
            const uint32_t cnt = min((uint32_t)nb, hi - k0);
            uint32_t bytes = 0;
            const float *src_host = nullptr;
            uint32_t slot = EMPTY;
            float *dst_host = nullptr;
            if ((uint32_t)lane < cnt) {
                const uint32_t item = k0 + lane;
                const int tl = find_table(s_pref, tcount, item);
                const int t = t0 + tl;
                const size_t kk = (size_t)t * g.n + (item - s_pref[tl]);
                slot = A.bb.fill_slot[kk];
                const uint32_t x = A.bb.fill_row[kk], o = A.bb.evict_row[kk];
                src_host = A.host[t] + (size_t)x * g.D;
                dst_host = o != EMPTY ? A.host[t] + (size_t)o * g.D : nullptr;
                bytes = rowb * (dst_host ? 2u : 1u);
            }
            s_slot[s][lane] = slot;
            s_dst_host[s][lane] = dst_host;
            const uint32_t tot = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) mbar_expect_tx(&bar[s], tot);
            __syncwarp();
            if (slot != EMPTY) {
                if (dst_host) bulk_g2s(vbuf(s, lane), A.storage + (size_t)slot * g.D, rowb, &bar[s]);
                bulk_g2s(vbuf(s, lane) + rowb, src_host, rowb, &bar[s]);
            }
        };
        for (uint32_t r = 0; r < min((uint32_t)XS, nround); r++) issue(r);
        for (uint32_t r = 0; r < nround; r++) {
            const int s = (int)((phase_ctr + r) % XS);
            mbar_wait(&bar[s], ((phase_ctr + r) / XS) & 1u);
            const uint32_t slot = s_slot[s][lane];
            if (slot != EMPTY) {
                float *dh = s_dst_host[s][lane];
                if (dh) bulk_s2g(dh, vbuf(s, lane), rowb);
                bulk_s2g(A.storage + (size_t)slot * g.D, vbuf(s, lane) + rowb, rowb);
            }
            bulk_commit();
            if (r + XS < nround) {
                bulk_wait_read0();  // stage s has been read out: refill it
                __syncwarp();
                issue(r + XS);
            }
        }
        phase_ctr += nround;
        bulk_wait0();
        __syncwarp();
    }
    bulk_wait0();
    __threadfence_system();
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

// items per round: one per lane, bounded so that XS stages of (victim, fill)
// row pairs fit the shared-memory budget
int exchange_items_per_round(int D) {
    const size_t budget = 192 * 1024;
    const size_t per_item = (size_t)2 * D * 4 * XS;
    size_t nb = budget / per_item;
    if (nb > 32) nb = 32;
    if (nb < 1) nb = 1;
    return (int)nb;
}

size_t exchange_smem_bytes(int D) { return (size_t)exchange_items_per_round(D) * 2 * D * 4 * XS; }

cudaError_t configure_exchange_kernel(int D) {
    return cudaFuncSetAttribute(k_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)exchange_smem_bytes(D));
}

cudaError_t launch_exchange(const XferArgs &a, int ctas, cudaStream_t s) {
    const int grid = ctas > 0 ? ctas : 16;
    k_exchange<<<grid, 32, exchange_smem_bytes(a.g.D), s>>>(a, exchange_items_per_round(a.g.D));
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
