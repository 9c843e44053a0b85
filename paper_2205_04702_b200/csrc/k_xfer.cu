// k_xfer.cu — the GPU side of [Collect] / [Exchange] / [Insert] (PAPER.md
// P:688-704) and the end-of-run write-back.
//
// Direction by direction, on measurements of this platform (
// profiles/r01_host_tlb_microbench.txt, r01_tma_xfer_microbench*.txt):
//   host -> HBM  by default the CPU gather thread has copied the missed rows
//                into a contiguous pinned slot (A.in_stage); the kernel moves
//                that slot into the freed Storage slots.  GPU reads of random
//                host rows are bound by host-side address translation and
//                slow the concurrent Train kernels; with in_stage == nullptr
//                (SP_CPU_GATHER=0) the kernel pulls each row from its table.
//                Rows move as whole-row TMA bulk copies (cp.async.bulk, one
//                request per row) from a bounded grid of 16 one-warp CTAs.
//   HBM -> host  the same kernel writes the victims, contiguously, into a
//                pinned staging slot with their host addresses, raises a
//                pinned flag when the last CTA is done, and the CPU threads of
//                the transfer engine scatter them into the host tables.
//   for every fill k (slot s, missed row x, previous resident o) of Plan(b),
//   staging index i = prefix + k:
//       smem <- Storage[s], smem' <- in_stage[i] (or host[t][x])   (both land first)
//       wb_stage[i] <- smem      if o is valid (dirty victim)
//       Storage[s]  <- smem'     (the freed slot gets the missed row)
#include "sp_internal.cuh"

#include <algorithm>

namespace sp {

// Completion of Transfer(b) for the scatter thread: every CTA's staging stores
// (rows and their destination addresses) are made visible system-wide, then
// the last CTA to arrive writes the item count and raises the pinned flag
// (and resets the counter for the next use of this ring slot).
__device__ __forceinline__ void publish_staged(const XferArgs &A, unsigned long long nstaged) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned k = atomicAdd(A.done_ctr, 1u);
        if (k == gridDim.x - 1) {
            *A.done_ctr = 0u;
            *(volatile unsigned long long *)A.staged_cnt = nstaged;
            __threadfence_system();
            *(volatile unsigned long long *)A.staged = (unsigned long long)(A.b + 1);
        }
    }
}


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

// k_pullfill (one warp per CTA): per fill, the victim row
// (HBM) and the missed row (host, zero-copy) are brought into shared memory
// by cp.async.bulk, then stored by cp.async.bulk to the staging row (host,
// contiguous) and the slot (HBM).  A whole 256-B row moves as one bulk
// request instead of sixteen 16-B loads.  The flattened fill list is split
// into contiguous shares, one per CTA, moved in rounds of nb items (one per
// lane) through XS shared-memory stages.
#ifndef SP_XS
#define SP_XS 4  // shared-memory stages per transfer CTA (compile-time A/B)
#endif
constexpr int XS = SP_XS;

// BF (SP_FLAG_BF16, reading R28): Storage rows are bf16.  A stage then also
// holds the victims as loaded (bf16) and the new rows narrowed (bf16): after
// a round lands the warp widens the victims (exact) and rounds the new rows
// to nearest even, and the bulk stores take the converted copies.
template <bool BF>
__global__ void __launch_bounds__(32) k_pullfill(XferArgs A, int nb) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[XS];
    __shared__ uint32_t s_pref[65];
    __shared__ uint32_t s_slot[XS][32], s_stage[XS][32];
    __shared__ unsigned long long s_dst[XS][32];  // direct write-back: host row of each victim
    if (*A.err != NO_ERR) return;
    unsigned long long *spn = span_base(A.span, SPK_XFER, A.b);
    span_mark(spn, 0);
    const Geometry g = A.g;
    const uint32_t rowb = (uint32_t)g.D * 4u;        // fp32 row (host side)
    const uint32_t srowb = BF ? rowb / 2u : rowb;     // Storage row
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < XS; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase_ctr = 0;  // rounds issued so far over all stages (parity source)
    uint32_t base_t0 = 0;    // staging rows of the tables before t0
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.m, t0, tcount, s_pref);  // (32 threads: one warp)
        const uint32_t total = s_pref[tcount];
        // per stage: nb victim rows, then nb new rows (contiguous, so a gathered
        // round moves as one bulk copy each way)
        // stage s: [nb] victims (fp32), [nb] new rows (fp32); BF adds [nb]
        // victims as loaded and [nb] new rows narrowed (bf16 each)
        const size_t sstride = (size_t)nb * (BF ? 3 : 2) * rowb;
        auto vbuf = [&](int s, int i) { return sm + s * sstride + (size_t)i * rowb; };
        auto nbuf = [&](int s, int i) { return sm + s * sstride + ((size_t)nb + i) * rowb; };
        auto v16 = [&](int s, int i) { return sm + s * sstride + (size_t)2 * nb * rowb + (size_t)i * srowb; };
        auto n16 = [&](int s, int i) { return sm + s * sstride + (size_t)2 * nb * rowb + ((size_t)nb + i) * srowb; };
        auto vload = [&](int s, int i) { return BF ? v16(s, i) : vbuf(s, i); };  // victim as loaded from Storage
        auto nstore = [&](int s, int i) { return BF ? n16(s, i) : nbuf(s, i); };  // new row as stored
        const bool direct = A.wb_direct != 0;  // victims straight to their host rows
        // items [0, Kg) of this table group were gathered by the CPU into the
        // contiguous pinned slot, the rest [Kg, total) are pulled from their
        // host rows (hybrid split: the CPU gather and the GPU pull run
        // concurrently).  Every CTA takes a contiguous share of BOTH ranges and
        // runs its pulled rounds first, so all CTAs pull while the CPU gathers
        // and reach the gathered rows last.
        const uint32_t Kg = !A.in_stage ? 0u
                            : (A.gfrac_q16 >= 65536u ? total : (uint32_t)(((unsigned long long)total * A.gfrac_q16) >> 16));
        const uint32_t G = gridDim.x, Pn = total - Kg;
        const uint32_t pper = (Pn + G - 1) / G, gper = (Kg + G - 1) / G;
        const uint32_t plo = Kg + min(Pn, blockIdx.x * pper), phi = Kg + min(Pn, blockIdx.x * pper + pper);
        const uint32_t glo = min(Kg, blockIdx.x * gper), ghi = min(Kg, blockIdx.x * gper + gper);
        const uint32_t npr = phi > plo ? (phi - plo + nb - 1) / nb : 0u;
        const uint32_t nround = npr + (ghi > glo ? (ghi - glo + nb - 1) / nb : 0u);
        auto round_k0 = [&](uint32_t r) { return r < npr ? plo + r * nb : glo + (r - npr) * nb; };
        auto round_cnt = [&](uint32_t r) {
            const uint32_t k0 = round_k0(r);
            return min((uint32_t)nb, (r < npr ? phi : ghi) - k0);
        };
        auto round_gathered = [&](uint32_t r) {  // the whole round comes from the gathered slot
            return A.in_stage != nullptr && !A.diag_nowb && r >= npr;
        };
        bool waited = !(A.gwait && ghi > glo);
        auto wait_gathered = [&]() {
            // hybrid: this CTA reads gathered rows; wait (in-kernel, on the
            // pinned progress counter) until the CPU has gathered batch b
            if (waited) return;
            if (lane == 0)
                while (*(volatile const unsigned long long *)A.gwait < (unsigned long long)(A.b + 1)) __nanosleep(512);
            __syncwarp();
            __threadfence_system();
            waited = true;
        };
        auto issue = [&](uint32_t r) {
            const int s = (int)((phase_ctr + r) % XS);
            const uint32_t k0 = round_k0(r);
            const uint32_t cnt = round_cnt(r);
            if (round_gathered(r)) wait_gathered();
            uint32_t bytes = 0, slot = EMPTY, stage = EMPTY;
            const float *src_host = nullptr;
            if ((uint32_t)lane < cnt) {
                const uint32_t item = k0 + lane;
                const int tl = find_table(s_pref, tcount, item);
                const int t = t0 + tl;
                const size_t kk = (size_t)t * g.n + (item - s_pref[tl]);
                slot = A.bb.fill_slot[kk];
                src_host = item < Kg ? A.in_stage + (size_t)(base_t0 + item) * g.D  // CPU-gathered, contiguous
                                     : A.host[t] + (size_t)A.bb.fill_row[kk] * g.D;
                const uint32_t old = A.bb.evict_row[kk];
                if (old != EMPTY && !A.diag_nowb) stage = direct ? (uint32_t)t : base_t0 + item;
                // the scatter thread's work list: where the staged row goes
                // (direct: the kernel itself stores the row there -- every
                // victim, or the share wb_q16 of them picked by a fixed hash
                // of the item index; the CPU scatters the rest)
                const unsigned long long dst =
                    old != EMPTY ? (unsigned long long)(uintptr_t)(A.host[t] + (size_t)old * g.D) : 0ull;
                const bool dir = direct || ((item * 2654435761u) >> 16) < A.wb_q16;
                s_dst[s][lane] = dir ? dst : 0ull;
                if (!direct) A.wb_dst[base_t0 + item] = dir ? 0ull : dst;
                bytes = rowb + (stage != EMPTY ? srowb : 0u);
            }
            if ((uint32_t)lane >= cnt) s_dst[s][lane] = 0ull;
            s_slot[s][lane] = slot;
            s_stage[s][lane] = stage;
            const uint32_t tot = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) mbar_expect_tx(&bar[s], tot);
            __syncwarp();
            if (round_gathered(r)) {  // the round's new rows: contiguous bulk copies, from the
                             // DMA'd device copy where it reaches, else the pinned slot
                if (lane == 0 && cnt) {
                    const uint32_t i0 = base_t0 + k0;
                    const uint32_t nd = A.in_dev ? min(cnt, A.in_dev_rows > i0 ? A.in_dev_rows - i0 : 0u) : 0u;
                    if (nd) bulk_g2s(nbuf(s, 0), A.in_dev + (size_t)i0 * g.D, nd * rowb, &bar[s]);
                    if (cnt > nd)
                        bulk_g2s(nbuf(s, nd), A.in_stage + (size_t)(i0 + nd) * g.D, (cnt - nd) * rowb, &bar[s]);
                }
            } else if (slot != EMPTY) {
                bulk_g2s(nbuf(s, lane), src_host, rowb, &bar[s]);
            }
            if (slot != EMPTY && stage != EMPTY)
                bulk_g2s(vload(s, lane), reinterpret_cast<const char *>(A.storage) + (size_t)slot * srowb, srowb, &bar[s]);
        };
        for (uint32_t r = 0; r < min((uint32_t)XS, nround); r++) issue(r);
        for (uint32_t r = 0; r < nround; r++) {
            const int s = (int)((phase_ctr + r) % XS);
            mbar_wait(&bar[s], ((phase_ctr + r) / XS) & 1u);
            if constexpr (BF) {
                // widen the victims, round the new rows (lanes stride over the
                // round's rows, four columns at a time); the bulk stores below
                // read the results through the async proxy
                const uint32_t cnt = round_cnt(r), D4 = (uint32_t)g.D / 4u;
                const float4 *n32 = reinterpret_cast<const float4 *>(nbuf(s, 0));
                const uint2 *v16r = reinterpret_cast<const uint2 *>(v16(s, 0));
                float4 *v32 = reinterpret_cast<float4 *>(vbuf(s, 0));
                uint2 *n16r = reinterpret_cast<uint2 *>(n16(s, 0));
                // rows are contiguous in each area: element e = row * D4 + c
#pragma unroll 4
                for (uint32_t e = lane; e < cnt * D4; e += 32) {
                    const float4 x = n32[e];
                    const uint2 y = v16r[e];
                    n16r[e] = SRow<true>::nar(x);
                    v32[e] = SRow<true>::wid(y);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
            }
            const uint32_t slot = s_slot[s][lane], stage = s_stage[s][lane];
            const unsigned long long dd = s_dst[s][lane];
            // victims written back by the kernel: one bulk store per row into
            // its host row
            if (slot != EMPTY && stage != EMPTY && dd) bulk_s2g(reinterpret_cast<void *>((uintptr_t)dd), vbuf(s, lane), rowb);
            if (direct) {
            } else if (round_gathered(r)) {
                // victims: one contiguous bulk store of the round's staging rows
                // (rows of fills without a victim carry garbage; their work-list
                // entry is 0, so the scatter skips them)
                const uint32_t k0 = round_k0(r), cnt = round_cnt(r);
                if (lane == 0 && cnt) bulk_s2g(A.wb_stage + (size_t)(base_t0 + k0) * g.D, vbuf(s, 0), cnt * rowb);
            } else if (slot != EMPTY && stage != EMPTY && !dd) {
                bulk_s2g(A.wb_stage + (size_t)stage * g.D, vbuf(s, lane), rowb);
            }
            if (slot != EMPTY) bulk_s2g(reinterpret_cast<char *>(A.storage) + (size_t)slot * srowb, nstore(s, lane), srowb);
            bulk_commit();
            if (r + XS < nround) {
                bulk_wait_read0();  // stage s has been read out: refill it
                __syncwarp();
                issue(r + XS);
            }
        }
        phase_ctr += nround;
        base_t0 += total;
        bulk_wait0();
        __syncwarp();
    }
    bulk_wait0();
    publish_staged(A, base_t0);  // base_t0 = sum over tables of m[t]
    span_mark(spn, 1);
}

// k_xfer_warp: the same Collect / Exchange / Insert work as k_pullfill with
// plain 16-B loads and stores from many warps instead of TMA bulk copies from
// a few.  Measured on this platform (profiles/r02_host_xlat_microbench.txt,
// r02_host_mix_microbench.txt): random 512-B host rows cost ~16 ns each on
// the GPU side whatever the page size, once >= ~600 warps have a row in
// flight (26 ns from 128 warps), and pulls and write-backs share that one
// limit; the CPU's row copies do not touch it.  So the kernel keeps one or
// two rows in flight per warp over a grid of ~600 warps, and the victims it
// does not write back itself go contiguously to pinned staging for the CPU
// scatter threads.  Per fill k (slot s, missed row x, previous resident o):
//     v = Storage[s] (if o valid);  r = host[t][x] (or the CPU-gathered row)
//     victim v -> its host row (share wbq of the valid victims, direct) or
//                 staging[k] + its host address in the scatter work list
//     Storage[s] = r
// Items run pulled-first; a warp reaching CPU-gathered items (hybrid) waits
// on the gather counter there.  Completion: publish_staged (last CTA).
template <int VPL>
__global__ void __launch_bounds__(128) k_xfer_warp(XferArgs A) {
    __shared__ uint32_t s_pref[65];
    if (*A.err != NO_ERR) return;
    unsigned long long *spn = span_base(A.span, SPK_XFER, A.b);
    span_mark(spn, 0);
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const long long W = (long long)gridDim.x * (blockDim.x / 32);
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    uint32_t base_t0 = 0;
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.m, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        const uint32_t Kg = !A.in_stage ? 0u
                            : (A.gfrac_q16 >= 65536u ? total : (uint32_t)(((unsigned long long)total * A.gfrac_q16) >> 16));
        bool waited = A.gwait == nullptr;
        // pulled items [Kg, total) first, then the CPU-gathered [0, Kg)
        for (long long j = gw; j < total; j += W) {
            const uint32_t item = (uint32_t)((j + Kg) % total);
            const bool gathered = item < Kg;
            if (gathered && !waited) {
                if (lane == 0)
                    while (*(volatile const unsigned long long *)A.gwait < (unsigned long long)(A.b + 1)) __nanosleep(256);
                __syncwarp();
                __threadfence_system();
                waited = true;
            }
            const int tl = find_table(s_pref, tcount, item);
            const int t = t0 + tl;
            const size_t kk = (size_t)t * g.n + (item - s_pref[tl]);
            const uint32_t slot = A.bb.fill_slot[kk], row = A.bb.fill_row[kk], old = A.bb.evict_row[kk];
            const bool victim = old != EMPTY && !A.diag_nowb;
            const float4 *src = reinterpret_cast<const float4 *>(
                gathered ? A.in_stage + (size_t)(base_t0 + item) * g.D : A.host[t] + (size_t)row * g.D);
            float4 v[VPL], r[VPL];
#pragma unroll
            for (int q = 0; q < VPL; q++) {
                const int c = lane + 32 * q;
                if (c < D4) {
                    if (victim) v[q] = st[(size_t)slot * D4 + c];
                    r[q] = __ldcv(src + c);  // (host memory: no stale L2 lines)
                }
            }
            // direct write-back for a share of the victims (a fixed hash of
            // the item index, so the CPU and GPU shares are spread evenly)
            const bool direct = victim && ((item * 2654435761u) >> 16) < A.wb_q16;
            float4 *dst = victim ? reinterpret_cast<float4 *>(A.host[t] + (size_t)old * g.D) : nullptr;
            float4 *stg = reinterpret_cast<float4 *>(A.wb_stage + (size_t)(base_t0 + item) * g.D);
#pragma unroll
            for (int q = 0; q < VPL; q++) {
                const int c = lane + 32 * q;
                if (c < D4) {
                    if (victim) {
                        if (direct) dst[c] = v[q];
                        else stg[c] = v[q];
                    }
                    st[(size_t)slot * D4 + c] = r[q];
                }
            }
            if (lane == 0)
                A.wb_dst[base_t0 + item] = (victim && !direct) ? (unsigned long long)(uintptr_t)dst : 0ull;
        }
        base_t0 += total;
        __syncthreads();  // (s_pref is reloaded for the next group)
    }
    publish_staged(A, base_t0);
    span_mark(spn, 1);
}

int pullfill_tma_items(int D, bool bf16) {
    const size_t budget = 192 * 1024, per_item = (size_t)(bf16 ? 3 : 2) * D * 4 * XS;
    size_t nb = budget / per_item;
    return (int)(nb > 32 ? 32 : (nb < 1 ? 1 : nb));
}

// sp_prefill (slots == rows for every table): slot slot_base[t] + id holds
// row id of table t; Storage itself is filled by a contiguous H2D copy
__global__ void __launch_bounds__(256) k_prefill_map(const uint32_t *slot_base, const unsigned long long *row_off,
                                                     int T, long long S_total, uint32_t *resident, uint32_t *hitmap) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < S_total;
         s += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = T;  // slot_base[lo] <= s < slot_base[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((long long)slot_base[mid] <= s) lo = mid;
            else hi = mid;
        }
        const uint32_t id = (uint32_t)(s - slot_base[lo]);
        resident[s] = id;
        hitmap[row_off[lo] + id] = (uint32_t)s;
    }
}

cudaError_t launch_prefill_map(const uint32_t *slot_base, const unsigned long long *row_off, int T,
                               long long S_total, uint32_t *resident, uint32_t *hitmap, cudaStream_t s) {
    k_prefill_map<<<148 * 8, 256, 0, s>>>(slot_base, row_off, T, S_total, resident, hitmap);
    return cudaGetLastError();
}

// initial class-0 log of every table: its slots in ascending order, all
// vacant (stamp VACANT), at log_base0[t]
__global__ void __launch_bounds__(256) k_log_init(const uint32_t *slot_base, const unsigned long long *log_base0,
                                                  int T, long long S_total, uint32_t *log_slot, int32_t *log_stamp) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < S_total;
         s += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = T;  // slot_base[lo] <= s < slot_base[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((long long)slot_base[mid] <= s) lo = mid;
            else hi = mid;
        }
        const size_t ix = (size_t)(log_base0[lo] + (unsigned long long)(s - slot_base[lo]));
        log_slot[ix] = (uint32_t)s;
        log_stamp[ix] = VACANT;
    }
}

cudaError_t launch_log_init(const uint32_t *slot_base, const unsigned long long *log_base0, int T, long long S_total,
                            uint32_t *log_slot, int32_t *log_stamp, cudaStream_t s) {
    k_log_init<<<148 * 8, 256, 0, s>>>(slot_base, log_base0, T, S_total, log_slot, log_stamp);
    return cudaGetLastError();
}

// Ragged bags (sp_plan_csr, reading R27): CSR (values, offsets [T*N+1]) ->
// the padded [T][N][L] index layout, -1 in positions past a bag's end.  One
// thread per (bag, position); offsets were validated on the host.
__global__ void __launch_bounds__(256) k_csr_pad(const long long *values, const long long *offsets, long long nbags,
                                                 int L, void *out, int out_i32) {
    const long long total = nbags * L;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long bag = i / L;
        const int p = (int)(i - bag * L);
        const long long o = __ldg(offsets + bag) + p;
        const long long id = o < __ldg(offsets + bag + 1) ? __ldg(values + o) : -1ll;
        if (out_i32) static_cast<int32_t *>(out)[i] = (int32_t)id;
        else static_cast<long long *>(out)[i] = id;
    }
}

cudaError_t launch_csr_pad(const long long *values, const long long *offsets, long long nbags, int L, void *out,
                           int out_i32, cudaStream_t s) {
    long long blocks = (nbags * L + 255) / 256;
    const long long cap = (long long)device_sms() * 8;
    k_csr_pad<<<(int)std::max(1ll, std::min(blocks, cap)), 256, 0, s>>>(values, offsets, nbags, L, out, out_i32);
    return cudaGetLastError();
}

// write back every resident slot (sp_flush); BF: bf16 rows widened (exact)
template <bool BF>
__global__ void __launch_bounds__(256) k_flush(FlushArgs A) {
    using SR = SRow<BF>;
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
        const typename SR::V *src = reinterpret_cast<const typename SR::V *>(A.storage) + (size_t)s * D4;
        for (int c = lane; c < D4; c += 32) dst[c] = SR::wid(src[c]);
    }
}

cudaError_t launch_xfer_warp(const XferArgs &a, int ctas, cudaStream_t s) {
    const int D4 = a.g.D / 4, g = ctas > 0 ? ctas : device_sms();
    if (D4 <= 32) k_xfer_warp<1><<<g, 128, 0, s>>>(a);
    else if (D4 <= 64) k_xfer_warp<2><<<g, 128, 0, s>>>(a);
    else if (D4 <= 128) k_xfer_warp<4><<<g, 128, 0, s>>>(a);
    else k_xfer_warp<8><<<g, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pullfill(const XferArgs &a, int ctas, cudaStream_t s) {
    const bool bf = a.g.bf16 != 0;
    const int nb = pullfill_tma_items(a.g.D, bf);
    const size_t smem = (size_t)nb * (bf ? 3 : 2) * a.g.D * 4 * XS;
    if (bf) k_pullfill<true><<<ctas > 0 ? ctas : 16, 32, smem, s>>>(a, nb);
    else k_pullfill<false><<<ctas > 0 ? ctas : 16, 32, smem, s>>>(a, nb);
    return cudaGetLastError();
}

// fp32 rows (device or mapped host memory) -> bf16 Storage rows, rounded to
// nearest even (SP_FLAG_BF16: sp_prefill, sp_pin_rows)
__global__ void __launch_bounds__(256) k_rows_to_bf16(const float4 *src, uint2 *dst, long long n4) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        dst[i] = SRow<true>::nar(src[i]);
}

cudaError_t launch_rows_to_bf16(const float *src, void *dst, long long count, int D, cudaStream_t s) {
    const long long n4 = count * (D / 4);
    if (n4 <= 0) return cudaSuccess;
    const long long blocks = (n4 + 255) / 256, cap = (long long)device_sms() * 8;
    k_rows_to_bf16<<<(int)std::min(blocks, cap), 256, 0, s>>>(reinterpret_cast<const float4 *>(src),
                                                               static_cast<uint2 *>(dst), n4);
    return cudaGetLastError();
}

cudaError_t launch_flush(const FlushArgs &a, cudaStream_t s) {
    long long blocks = ((long long)a.S_total + 7) / 8;
    long long cap = (long long)device_sms() * 8;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    if (a.g.bf16) k_flush<true><<<grid, 256, 0, s>>>(a);
    else k_flush<false><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

// attributes of the transfer kernel on the current device (sp_create; kernel
// attributes are per device, so every context sets them on its own GPU)
cudaError_t configure_xfer_kernels() {
    apply_carveout(k_pullfill<false>);
    apply_carveout(k_pullfill<true>);
    cudaFuncSetAttribute(k_pullfill<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
    return cudaFuncSetAttribute(k_pullfill<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
}

}  // namespace sp
