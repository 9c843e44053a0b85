// k_train.cu — the [Training] stage's embedding part on the scratchpad
// (forward, MLP, backward and update as ONE stage so that
// RAW-1 is honoured).  Every access is a scratchpad hit by construction.
//
//   k_fwd   EmbeddingBag forward: pooled[t][s] = sum over p of
//           Storage[slot(t,s,p)], fp32 left fold in ascending p.  HBM-bound:
//           one 16-byte vector per lane, a lane group of D/4 lanes per bag,
//           all L row loads of a bag issued before the fold.
//   k_bwd   gradient duplication + coalescing fused with the SGD
//           update: per unique row, the gradients of its
//           occurrences (contiguous in the sorted occurrence list built at
//           dedup) are summed in fp64 and the row is updated in place,
//           w = fmaf(-lr, (float)sum, w).  One owner per unique row -> no
//           atomics on Storage.  Hot (Zipf-head) rows are folded by a whole
//           CTA with a fixed tree; the rest by one lane group each.
//   k_surrogate  the harness's MLP stand-in g = fmaf(gamma, pooled, delta).
#include "sp_internal.cuh"

#include <cuda.h>  // CUtensorMap (tile::gather4)

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace sp {

namespace {

template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G >= 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
    }
}


__device__ __forceinline__ void add4(float4 &a, const float4 &b) {
    a.x = a.x + b.x; a.y = a.y + b.y; a.z = a.z + b.z; a.w = a.w + b.w;
}

}  // namespace

// ---------------------------------------------------------------- forward
// G lanes per bag, VPL float4 per lane (D/4 = G*VPL).  A lane group folds BU
// bags at a time (bags g, g+S, ..., S = all groups of the grid): their slot
// indices, then their rows for lookup position p, are all in flight together,
// so even L = 1 (one row per bag) keeps BU rows per group outstanding.  Each
// bag is still a left fold in ascending p (bit-exact with the oracle).
constexpr int FWD_ROUNDS = 4;  // k_fwd dynamic chunks: rounds per claim
template <int G, int VPL, bool PAD, bool BF>
__device__ __forceinline__ void fwd_body(const TrainArgs &A) {
    using SR = SRow<BF>;  // fp32 or bf16 Storage rows (R28: widened, folded in fp32)
    // (no work after a latched error, but the dynamic path still counts its
    // warps out so the claim counters reset)
    const bool dead = *A.err != NO_ERR;
    if (dead && (PAD || !A.fctr)) return;
    constexpr int BU = VPL >= 4 ? 1 : (VPL == 2 ? 2 : 4);
    const int L = A.g.L, D4 = A.g.D / 4;
    const long long nbags = dead ? 0 : (long long)A.g.T * A.g.N;
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    const typename SR::V *st = reinterpret_cast<const typename SR::V *>(A.storage) + lane;
    float4 *out = reinterpret_cast<float4 *>(A.pooled) + lane;
    const long long S = (long long)gridDim.x * gpb;
    if constexpr (PAD) {
        // ragged bags (-1 padding, reading R27): a padded position has slot
        // EMPTY and is skipped; a bag with no lookup pools to zeros; the fold
        // starts from the first real row (as the oracle's)
        for (long long bag = (long long)blockIdx.x * gpb + threadIdx.x / G; bag < nbags; bag += S) {
            const uint32_t *so = A.bb.slot_of_occ + bag * L;
            float4 acc[VPL];
            bool first = true;
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int p = 0; p < L; p++) {
                const uint32_t sl = __ldg(so + p);
                if (sl == EMPTY) continue;
#pragma unroll
                for (int v = 0; v < VPL; v++) {
                    const float4 r = SR::wid(__ldg(st + (size_t)sl * D4 + v * G));
                    if (first) acc[v] = r;
                    else add4(acc[v], r);
                }
                first = false;
            }
#pragma unroll
            for (int v = 0; v < VPL; v++) __stcs(out + bag * D4 + v * G, acc[v]);
        }
        return;
    } else {
    // BU bags of the lane group in flight: bag0, bag0 + S, ..., bag0 + (BU-1)*S
    auto bags = [&](long long bag0, long long S) {
        const uint32_t *so[BU];
        bool ok[BU];
        float4 acc[BU][VPL];
#pragma unroll
        for (int u = 0; u < BU; u++) {
            const long long bag = bag0 + u * S;
            ok[u] = bag < nbags;
            so[u] = A.bb.slot_of_occ + (ok[u] ? bag : 0) * L;
        }
        uint32_t s[BU];
#pragma unroll
        for (int u = 0; u < BU; u++) s[u] = __ldg(so[u]);
#pragma unroll
        for (int u = 0; u < BU; u++)
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[u][v] = SR::wid(__ldg(st + (size_t)s[u] * D4 + v * G));
        for (int p = 1; p < L; p++) {
#pragma unroll
            for (int u = 0; u < BU; u++) s[u] = __ldg(so[u] + p);
            float4 r[BU][VPL];
#pragma unroll
            for (int u = 0; u < BU; u++)
#pragma unroll
                for (int v = 0; v < VPL; v++) r[u][v] = SR::wid(__ldg(st + (size_t)s[u] * D4 + v * G));
#pragma unroll
            for (int u = 0; u < BU; u++)
#pragma unroll
                for (int v = 0; v < VPL; v++) add4(acc[u][v], r[u][v]);
        }
#pragma unroll
        for (int u = 0; u < BU; u++)
            if (ok[u])
#pragma unroll
                for (int v = 0; v < VPL; v++) __stcs(out + (bag0 + u * S) * D4 + v * G, acc[u][v]);
    };
    if (!A.fctr) {  // static grid stride (SP_FWD_DYN=0)
        for (long long bag0 = (long long)blockIdx.x * gpb + threadIdx.x / G; bag0 < nbags; bag0 += BU * S) bags(bag0, S);
        return;
    }
    // dynamic: a warp takes chunks of WB consecutive bags (FWD_ROUNDS rounds
    // of its 32/G lane groups x BU bags), the first by its index, the rest
    // claimed from one of TCTR_GROUPS counters (claim issued one chunk ahead),
    // so warps that become resident late (SMs shared with k_push / k_pullfill)
    // take fewer bags; the last warp out resets the counters
    constexpr int GPW = 32 / G, WB = GPW * BU * FWD_ROUNDS;
    const int lw = threadIdx.x & 31, gw = lw / G;
    const long long nch = (nbags + WB - 1) / WB;
    const long long W = (long long)gridDim.x * (blockDim.x >> 5);
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t *ctrs = A.fctr + (size_t)(A.span_b % RING) * TCTR_STRIDE;
    const int grp = (int)(wid % TCTR_GROUPS);
    for (long long ch = wid; ch < nch;) {
        uint32_t claim = 0;
        if (lw == 0) claim = atomicAdd(ctrs + grp * 32, 1u);
#pragma unroll 1
        for (int r = 0; r < FWD_ROUNDS; r++) bags(ch * WB + (long long)r * GPW * BU + gw, GPW);
        ch = W + grp + (long long)TCTR_GROUPS * __shfl_sync(0xffffffffu, claim, 0);
    }
    if (lw == 0 && atomicAdd(ctrs + TCTR_GROUPS * 32, 1u) == (uint32_t)(W - 1))
        for (int j = 0; j <= TCTR_GROUPS; j++) ctrs[j * 32] = 0u;
    }
}

template <int G, int VPL>
__global__ void __launch_bounds__(256) k_fwd(TrainArgs A) {
    unsigned long long *sp = span_base(A.span, SPK_FWD, A.span_b);
    span_mark(sp, 0);
    fwd_body<G, VPL, false, false>(A);
    if (sp) {
        __syncthreads();
        span_mark(sp, 1);
    }
}
// ragged bags (SP_FLAG_PADDING): its own instance keeps the fixed-L kernel lean
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_fwd_pad(TrainArgs A) {
    unsigned long long *sp = span_base(A.span, SPK_FWD, A.span_b);
    span_mark(sp, 0);
    fwd_body<G, VPL, true, false>(A);
    if (sp) {
        __syncthreads();
        span_mark(sp, 1);
    }
}

// generic D (D/4 not a power-of-two multiple of 32): 32 lanes, strided columns
template <bool BF>
__device__ __forceinline__ void fwd_generic_body(const TrainArgs &A) {
    using SR = SRow<BF>;
    if (*A.err != NO_ERR) return;
    const int L = A.g.L, D4 = A.g.D / 4;
    const long long nbags = (long long)A.g.T * A.g.N;
    const int lane = threadIdx.x & 31;
    const typename SR::V *st = reinterpret_cast<const typename SR::V *>(A.storage);
    float4 *out = reinterpret_cast<float4 *>(A.pooled);
    for (long long bag = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; bag < nbags;
         bag += (long long)gridDim.x * (blockDim.x / 32)) {
        const uint32_t *so = A.bb.slot_of_occ + bag * L;
        for (int c = lane; c < D4; c += 32) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            bool first = true;
            for (int p = 0; p < L; p++) {
                const uint32_t sl = __ldg(so + p);
                if (sl == EMPTY) continue;  // padding (reading R27)
                const float4 r = SR::wid(__ldg(st + (size_t)sl * D4 + c));
                if (first) acc = r;
                else add4(acc, r);
                first = false;
            }
            out[bag * D4 + c] = acc;
        }
    }
}

__global__ void __launch_bounds__(256) k_fwd_generic(TrainArgs A) { fwd_generic_body<false>(A); }
__global__ void __launch_bounds__(256) k_fwd_pad_generic(TrainArgs A) { fwd_generic_body<false>(A); }
__global__ void __launch_bounds__(256) k_fwd_bf_generic(TrainArgs A) { fwd_generic_body<true>(A); }
__global__ void __launch_bounds__(256) k_fwd_pad_bf_generic(TrainArgs A) { fwd_generic_body<true>(A); }
// bf16 Storage instances (SP_FLAG_BF16)
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_fwd_bf(TrainArgs A) {
    unsigned long long *sp = span_base(A.span, SPK_FWD, A.span_b);
    span_mark(sp, 0);
    fwd_body<G, VPL, false, true>(A);
    if (sp) {
        __syncthreads();
        span_mark(sp, 1);
    }
}
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_fwd_pad_bf(TrainArgs A) {
    unsigned long long *sp = span_base(A.span, SPK_FWD, A.span_b);
    span_mark(sp, 0);
    fwd_body<G, VPL, true, true>(A);
    if (sp) {
        __syncthreads();
        span_mark(sp, 1);
    }
}

// --------------------------------------------------------------- backward
struct Acc4 { double x, y, z, w; };

__device__ __forceinline__ void acc_add(Acc4 &a, const float4 &g) {
    a.x += (double)g.x; a.y += (double)g.y; a.z += (double)g.z; a.w += (double)g.w;
}

__device__ __forceinline__ float4 sgd(const float4 &w, const Acc4 &a, float lr) {
    float4 r;
    r.x = fmaf(-lr, (float)a.x, w.x);
    r.y = fmaf(-lr, (float)a.y, w.y);
    r.z = fmaf(-lr, (float)a.z, w.z);
    r.w = fmaf(-lr, (float)a.w, w.w);
    return r;
}

__device__ __forceinline__ float4 sgd32(const float4 &w, const float4 &g, float lr) {
    return make_float4(fmaf(-lr, g.x, w.x), fmaf(-lr, g.y, w.y), fmaf(-lr, g.z, w.z), fmaf(-lr, g.w, w.w));
}

__device__ __forceinline__ double4 ldcg_d4(const double4 *p) {  // L2 (written by other SMs)
    const double2 lo = __ldcg(reinterpret_cast<const double2 *>(p));
    const double2 hi = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(lo.x, lo.y, hi.x, hi.y);
}

__device__ __forceinline__ double4 shfl_xor_d4(const double4 &v, int m) {
    return make_double4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                        __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
}

// tuning knobs (measured defaults; -D overrides for A/B builds)
#ifndef SP_BWD_RB
#define SP_BWD_RB 4   // D <= 128: gradient rows of a hot segment in flight per lane group
#endif
#ifndef SP_BWD_RQ
#define SP_BWD_RQ 4   // D <= 128: chunk records folded together per lane group
#endif
#ifndef SP_BWD_MINB
#define SP_BWD_MINB 2 // resident CTAs per SM the register budget is sized for
#endif

// Warp-centric: every work item belongs to one warp (hot-row segment) or one
// lane group of G lanes (chunk records), so there is no block barrier after
// the prologue and every warp keeps several rows in flight.
//  H  hot-row segment (<= hs occurrences of a Zipf-head row): the warp's NG
//     lane groups take occurrences g, g+NG, ... (RB rows in flight each) and
//     accumulate in fp64; a fixed xor tree over the groups gives the segment
//     sum.  A single-segment row is updated at once; otherwise the segment
//     writes an fp64 partial and the last segment to arrive (counter per row)
//     folds the partials in segment order and applies SGD.  Every fold order
//     depends only on the row's occurrence count.
//  N  chunk records (<= CH occurrences, bag ids inline): BU records per lane
//     group at once -- headers, Storage rows and the gradient rows of their
//     first two occurrences all in flight together.  A record of <= 2
//     occurrences is summed in fp32, which equals the fp32 rounding of the
//     exact (fp64) sum (reading R7: two fp32 values sum exactly in fp64, or
//     the smaller is below half an ulp of the larger); longer ones continue
//     in fp64 in ascending occurrence order.  One owner per unique row: no
//     atomics on Storage.
template <int G, int VPL>
__global__ void __launch_bounds__(256, SP_BWD_MINB) k_bwd(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    constexpr int NG = 32 / G;                                 // lane groups per warp
    constexpr int RB = VPL >= 4 ? 1 : (VPL == 2 ? 2 : SP_BWD_RB);  // hot rows in flight per group
    __shared__ uint32_t s_ph[65], s_pc[65];
    const int lane = threadIdx.x % G;
    const int grp = (threadIdx.x & 31) / G;
    const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const long long W = (long long)gridDim.x * (blockDim.x / 32);
    const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    const bool one_group = g.T <= 64;
    if (one_group) table_prefix2(A.bb.nhot, A.bb.nchunks, 0, g.T, s_ph, s_pc);
    griddep_wait();  // (PDL) the surrogate's gradients are complete from here on
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        if (!one_group) table_prefix2(A.bb.nhot, A.bb.nchunks, t0, tcount, s_ph, s_pc);
        const uint32_t Ht = (A.diag & 8) ? 0u : s_ph[tcount], Ct = (A.diag & 16) ? 0u : s_pc[tcount];
        // ---- H: one warp per hot-row segment
        for (long long item = gw; item < Ht; item += W) {
            const int tl = find_table(s_ph, tcount, (uint32_t)item);
            const int t = t0 + tl;
            const uint32_t h = (uint32_t)item - s_ph[tl];
            const uint4 hr = A.bb.hot_rec[(size_t)t * g.nh + h];
            const uint32_t slot = hr.x, lo = hr.y, len = hr.z & HOT_LEN_MASK, k = hr.w, nseg = hr.z >> HOT_LEN_BITS;
            const uint32_t *occ = A.bb.sorted_occ + (size_t)t * g.n + lo;
            const float4 *gb = grad + (size_t)t * g.N * D4 + lane;
            Acc4 acc[VPL];
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[v] = Acc4{0.0, 0.0, 0.0, 0.0};
            for (uint32_t k0 = grp; k0 < len; k0 += NG * RB) {
                float4 r[RB][VPL];
#pragma unroll
                for (int q = 0; q < RB; q++) {
                    const uint32_t kq = k0 + (uint32_t)q * NG;
                    if (kq < len) {
                        const uint32_t bag = __ldg(occ + kq) / (uint32_t)g.L;
#pragma unroll
                        for (int v = 0; v < VPL; v++) r[q][v] = __ldg(gb + (size_t)bag * D4 + v * G);
                    }
                }
#pragma unroll
                for (int q = 0; q < RB; q++)
                    if (k0 + (uint32_t)q * NG < len)
#pragma unroll
                        for (int v = 0; v < VPL; v++) acc_add(acc[v], r[q][v]);
            }
            // fixed xor tree over the warp's lane groups: every group ends
            // with the segment sum (order fixed by NG only)
#pragma unroll
            for (int v = 0; v < VPL; v++) {
                double4 m = make_double4(acc[v].x, acc[v].y, acc[v].z, acc[v].w);
#pragma unroll
                for (int o = G; o < 32; o <<= 1) {
                    const double4 p = shfl_xor_d4(m, o);
                    m.x += p.x; m.y += p.y; m.z += p.z; m.w += p.w;
                }
                acc[v] = Acc4{m.x, m.y, m.z, m.w};
            }
            if (nseg == 1) {
                if (grp == 0)
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        float4 *wp = st + (size_t)slot * D4 + lane + v * G;
                        *wp = sgd(*wp, acc[v], A.lr);
                    }
                continue;
            }
            // several segments: fp64 partials meet in a two-level fixed tree --
            // the last of each group of 8 consecutive segments folds the
            // group's partials in order, the last group folds the group sums in
            // order and applies SGD (the shape depends only on nseg)
            double *prow = A.partial + ((size_t)t * g.nh + (h - k)) * g.D;  // segment 0 of the row
            uint32_t *cnt = A.bb.hot_cnt + (size_t)t * g.nh + (h - k);
            if (grp == 0)
#pragma unroll
                for (int v = 0; v < VPL; v++)
                    reinterpret_cast<double4 *>(prow + (size_t)k * g.D)[lane + v * G] =
                        make_double4(acc[v].x, acc[v].y, acc[v].z, acc[v].w);
            const uint32_t ng = (nseg + 7u) / 8u, grpi = k / 8u, gsz = min(8u, nseg - 8u * grpi);
            auto arrive = [&](uint32_t *ctr, uint32_t total) {
                __threadfence();
                __syncwarp();
                uint32_t last = 0;
                if ((threadIdx.x & 31) == 0) last = atomicAdd(ctr, 1u) == total - 1u;
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) __threadfence();
                return last != 0;
            };
            // fold `count` partials at stride `step` segments from `first` (lane l: float4 columns l, l+32, ...)
            auto fold = [&](uint32_t first, uint32_t count, uint32_t step, int col) {
                const double4 *p0 = reinterpret_cast<const double4 *>(prow) + col;
                double4 m = make_double4(0.0, 0.0, 0.0, 0.0);
                uint32_t q = 0;
                for (; q + 2 <= count; q += 2) {
                    double4 x[2];
#pragma unroll
                    for (int u = 0; u < 2; u++) x[u] = ldcg_d4(p0 + (size_t)(first + (q + u) * step) * D4);
#pragma unroll
                    for (int u = 0; u < 2; u++) { m.x += x[u].x; m.y += x[u].y; m.z += x[u].z; m.w += x[u].w; }
                }
                for (; q < count; q++) {
                    const double4 x = ldcg_d4(p0 + (size_t)(first + q * step) * D4);
                    m.x += x.x; m.y += x.y; m.z += x.z; m.w += x.w;
                }
                return m;
            };
            if (ng > 1) {
                if (!arrive(cnt + 1 + grpi, gsz)) continue;
                for (int col = threadIdx.x & 31; col < D4; col += 32) {  // group sum -> its first segment's slot
                    const double4 m = fold(8u * grpi, gsz, 1u, col);
                    reinterpret_cast<double4 *>(prow + (size_t)(8u * grpi) * g.D)[col] = m;
                }
            }
            if (!arrive(cnt, ng > 1 ? ng : nseg)) continue;
            for (int col = threadIdx.x & 31; col < D4; col += 32) {
                const double4 m = ng > 1 ? fold(0u, ng, 8u, col) : fold(0u, nseg, 1u, col);
                float4 *wp = st + (size_t)slot * D4 + col;
                *wp = sgd(*wp, Acc4{m.x, m.y, m.z, m.w}, A.lr);
            }
        }
        // ---- N: chunk records in warp batches of 32: lane i loads the header
        // (slot, len, bag0, bag1) of record base+i in one coalesced read, then
        // each lane group folds RQ records per sub-round with every Storage
        // and gradient row of those records in flight together
        constexpr int RQ = VPL >= 4 ? 1 : (VPL == 2 ? 2 : SP_BWD_RQ);
        for (long long base = gw * 32; base < Ct; base += W * 32) {
            uint4 myhd = make_uint4(0, 0, 0, 0);
            uint32_t mytt = 0, myci = 0;
            if (base + (threadIdx.x & 31) < Ct) {
                const uint32_t c = (uint32_t)(base + (threadIdx.x & 31));
                const int tl = find_table(s_pc, tcount, c);
                mytt = (uint32_t)(t0 + tl);
                myci = c - s_pc[tl];
                myhd = __ldg(reinterpret_cast<const uint4 *>(A.bb.chunk_rec + (size_t)mytt * g.nc + myci));
            }
            const uint32_t nrec = (uint32_t)min(32ll, Ct - base);
            uint32_t longm = 0;  // records (warp-batch index) with > 2 occurrences, folded below
            for (uint32_t j0 = 0; j0 < nrec; j0 += NG * RQ) {
                uint4 hd[RQ];
                uint32_t tt[RQ];
#pragma unroll
                for (int q = 0; q < RQ; q++) {
                    const int src = (int)(j0 + q * NG + grp);  // this group's q-th record of the sub-round
                    hd[q].x = __shfl_sync(0xffffffffu, myhd.x, src & 31);
                    hd[q].y = __shfl_sync(0xffffffffu, myhd.y, src & 31);
                    hd[q].z = __shfl_sync(0xffffffffu, myhd.z, src & 31);
                    hd[q].w = __shfl_sync(0xffffffffu, myhd.w, src & 31);
                    tt[q] = __shfl_sync(0xffffffffu, mytt, src & 31);
                    if (src >= (int)nrec) hd[q].y = 0u;
                }
                float4 w[RQ][VPL], g0[RQ][VPL], g1[RQ][VPL];
#pragma unroll
                for (int q = 0; q < RQ; q++) {
                    if (hd[q].y == 0u || hd[q].y > 2u) continue;
                    const float4 *gb = grad + (size_t)tt[q] * g.N * D4 + lane;
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        w[q][v] = st[(size_t)hd[q].x * D4 + lane + v * G];
                        g0[q][v] = __ldg(gb + (size_t)hd[q].z * D4 + v * G);
                        if (hd[q].y == 2u) g1[q][v] = __ldg(gb + (size_t)hd[q].w * D4 + v * G);
                    }
                }
#pragma unroll
                for (int q = 0; q < RQ; q++) {
                    const uint32_t len = hd[q].y;
                    if (len == 0u) continue;
                    if (len > 2u) {
                        longm |= 1u << (j0 + q * NG + grp);
                        continue;
                    }
                    float4 *wp = st + (size_t)hd[q].x * D4 + lane;
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        float4 sg = g0[q][v];
                        if (len == 2u) { sg.x += g1[q][v].x; sg.y += g1[q][v].y; sg.z += g1[q][v].z; sg.w += g1[q][v].w; }
                        wp[v * G] = sgd32(w[q][v], sg, A.lr);
                    }
                }
            }
            // > 2 occurrences (rare in the Zipf tail): fp64 in ascending
            // occurrence order, this group's own records of the batch.  Each
            // group marked only its own records: the union makes the loop
            // (and its full-warp shuffles) warp-uniform.
            longm = __reduce_or_sync(0xffffffffu, longm);
            while (longm) {
                const int i = __ffs(longm) - 1;
                longm &= longm - 1;
                const uint32_t slot = __shfl_sync(0xffffffffu, myhd.x, i);  // (every lane: uniform i)
                const uint32_t len = __shfl_sync(0xffffffffu, myhd.y, i);
                const uint32_t tu = __shfl_sync(0xffffffffu, mytt, i);
                const uint32_t cu = __shfl_sync(0xffffffffu, myci, i);
                if ((i % NG) != grp) continue;  // owned by another group of the warp
                const uint32_t *bags = A.bb.chunk_rec[(size_t)tu * g.nc + cu].bag;
                const float4 *gb = grad + (size_t)tu * g.N * D4 + lane;
                float4 *wp = st + (size_t)slot * D4 + lane;
                Acc4 acc[VPL];
#pragma unroll
                for (int v = 0; v < VPL; v++) acc[v] = Acc4{0.0, 0.0, 0.0, 0.0};
                for (uint32_t q0 = 0; q0 < len; q0 += 4) {
                    float4 r[4][VPL];
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (q0 + q < len) {
                            const uint32_t bag = __ldg(bags + q0 + q);
#pragma unroll
                            for (int v = 0; v < VPL; v++) r[q][v] = __ldg(gb + (size_t)bag * D4 + v * G);
                        }
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (q0 + q < len)
#pragma unroll
                            for (int v = 0; v < VPL; v++) acc_add(acc[v], r[q][v]);
                }
#pragma unroll
                for (int v = 0; v < VPL; v++) wp[v * G] = sgd(wp[v * G], acc[v], A.lr);
            }
        }
    }
}

// ------------------------------------------------ backward, tiled (default)
// The sorted occurrence list of each table (built at dedup: occurrences
// grouped by unique row, ascending within a row) is cut into fixed tiles of
// TR rows; one warp (one CTA) takes a tile at a time:
//   1. lane r reads sorted occurrence r of the tile and its unique (coalesced)
//      and issues ONE TMA bulk copy (cp.async.bulk) of that occurrence's
//      gradient row pooled_grad[t][occ / L] into shared memory; the first lane
//      of every row that lies wholly inside the tile also bulk-copies the
//      row's Storage row.  All of the tile's rows are in flight at once on
//      one mbarrier -- the memory-level parallelism comes from the copy
//      engine, not from registers.
//   2. the warp folds the tile's rows in order, lane c owning float4 column
//      c (+32, ...), in fp64 (reading R7).  At the end of a row wholly inside
//      the tile: w = fmaf(-lr, (float)sum, w) straight to Storage (the whole
//      row's sum in ascending occurrence order: the oracle's order).
//   3. a row spanning several tiles (the Zipf head) leaves one fp64 piece per
//      tile; the last piece to arrive (counter per row) folds the pieces in
//      tile order -- through a second level of groups of 8 pieces when there
//      are more than 8 -- and applies SGD.  The fold shape depends only on the
//      row's position in the sorted list, never on the grid.
// Every tile is the same size whatever the skew, so the grid is balanced by
// construction (no hot/cold work lists, no dynamic work counters); one owner
// per unique row, so no atomics on Storage.
namespace {
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool bar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void row_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
// TMA tile::gather4: rows r0..r3 (all D columns) of the 2-D tensor of `tm`
// into consecutive rows of shared memory at dst, completion on bar
__device__ __forceinline__ void rows4_g2s(void *dst, const CUtensorMap *tm, uint32_t r0, uint32_t r1, uint32_t r2,
                                          uint32_t r3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_addr(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_addr(bar))
        : "memory");
}
// 16-B async copy global -> shared (LDGSTS), L2 only
__device__ __forceinline__ void cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void dadd4(double4 &a, const double4 &b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
__device__ __forceinline__ double4 ld_piece(const double *p) {  // L2: written by other SMs
    return ldcg_d4(reinterpret_cast<const double4 *>(p));
}
// warp-wide "last of `total` arrivals at *ctr": the warp's writes are
// ordered before lane 0's acq_rel atomic by the warp barrier (release), and
// the winner's later reads after it (acquire) -- the semaphore pattern of
// CUTLASS's barrier, without a full fence (__threadfence costs MEMBAR +
// ERRBAR + CCTL: ~20% of k_bwd_tile's stall samples; SP_DIAG=256 restores it)
__device__ __forceinline__ bool warp_arrive_last(uint32_t *ctr, uint32_t total, bool full_fence) {
    if (full_fence) __threadfence();
    __syncwarp();
    uint32_t last = 0;
    if ((threadIdx.x & 31) == 0) {
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
        last = prev == total - 1u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    __syncwarp();
    if (last && full_fence) __threadfence();
    return last != 0;
}
}  // namespace

// 2.-3. of a tile (shared by k_bwd_tile and the warp-specialised k_bwd_ws):
// fold the staged rows segment by segment and update Storage, or leave the
// pieces of rows spanning tiles and fold them at the last arrival.  Lane
// masks: lmask = last row of each segment in the tile, wmask = first row of
// each row wholly inside it; per lane (row r): slot, uid.
template <int VPL, bool BF = false>
__device__ __forceinline__ void bwd_fold_tile(const TrainArgs &A, int t, int k, unsigned lmask, unsigned wmask,
                                              uint32_t slot, uint32_t uid, const float4 *sg,
                                              const typename SRow<BF>::V *sw, uint32_t eslo = EMPTY,
                                              uint32_t eshi = EMPTY) {
    // BF: Storage rows are bf16 (reading R28): widened on read, the update
    // rounded to nearest even on write; the sums are the same as for fp32
    using SR = SRow<BF>;
    // eslo / eshi: segment offsets of the row of lane 0 (and of the last
    // row, on its lane), prefetched with the tile's metadata; EMPTY = load here
    const Geometry &g = A.g;
    const int D4 = g.D / 4, TR = A.tr, NT = A.ntiles;
    const int lane = threadIdx.x & 31;
    typename SR::V *st = reinterpret_cast<typename SR::V *>(A.storage);
    const size_t tb = (size_t)t * g.n;
    // 2. fold segment by segment (a segment = one row's occurrences in
    // this tile).  A whole row of 1 or 2 occurrences is summed in fp32:
    // that is the fp32 rounding of the exact sum, i.e. the oracle's
    // (float)(fp64 sum) (reading R7); longer rows and pieces of rows
    // spanning tiles accumulate in fp64 in ascending occurrence order.
    // whole rows of one occurrence (the segment starts and ends on row r) and
    // of two (starts at r, ends at r+1) first, in straight loops: two
    // rows of each per trip, loads before stores (SP_DIAG=32 sends every row
    // through the fp64 path, A/B)
    const unsigned lone1 = (A.diag & 32) ? 0u : (wmask & lmask);
    const unsigned lone2 = (A.diag & 32) ? 0u : (wmask & (lmask >> 1) & ~lmask);
    auto wrow = [&](int r) { return A.g4 ? __popc(wmask & ((1u << r) - 1u)) : r; };  // its staged Storage row
    for (unsigned m1 = lone1; m1;) {
        const int ra = __ffs(m1) - 1;
        m1 &= m1 - 1;
        const int rb = m1 ? __ffs(m1) - 1 : -1;
        if (rb >= 0) m1 &= m1 - 1;
        const uint32_t sa = __shfl_sync(0xffffffffu, slot, ra), sb = __shfl_sync(0xffffffffu, slot, rb & 31);
        const int wa = wrow(ra), wb = rb >= 0 ? wrow(rb) : 0;
#pragma unroll
        for (int v = 0; v < VPL; v++) {
            const int c = lane + 32 * v;
            if (c < D4) {
                const float4 ga = sg[(size_t)ra * D4 + c], xa = SR::wid(sw[(size_t)wa * D4 + c]);
                float4 gb, xb;
                if (rb >= 0) { gb = sg[(size_t)rb * D4 + c]; xb = SR::wid(sw[(size_t)wb * D4 + c]); }
                st[(size_t)sa * D4 + c] = SR::nar(sgd32(xa, ga, A.lr));
                if (rb >= 0) st[(size_t)sb * D4 + c] = SR::nar(sgd32(xb, gb, A.lr));
            }
        }
    }
    for (unsigned m2 = lone2; m2; m2 &= m2 - 1) {
        const int r = __ffs(m2) - 1;
        const uint32_t s2 = __shfl_sync(0xffffffffu, slot, r);
        const int w2 = wrow(r);
#pragma unroll
        for (int v = 0; v < VPL; v++) {
            const int c = lane + 32 * v;
            if (c < D4) {
                float4 gs = sg[(size_t)r * D4 + c];
                add4(gs, sg[(size_t)(r + 1) * D4 + c]);
                st[(size_t)s2 * D4 + c] = SR::nar(sgd32(SR::wid(sw[(size_t)w2 * D4 + c]), gs, A.lr));
            }
        }
    }
    // the other segments: each ends at a bit of `ends`, starts after the
    // previous bit of lmask
    unsigned ends = lmask & ~(lone1 | (lone2 << 1));
    while (ends) {
        const int r1 = __ffs(ends) - 1;  // its last row
        ends &= ends - 1;
        const unsigned below = lmask & ((1u << r1) - 1u);
        const int r0 = below ? 32 - __clz(below) : 0;  // its first row
        const uint32_t s = __shfl_sync(0xffffffffu, slot, r0);
        const bool wh = (wmask >> r0) & 1u;
        const int wr = wrow(r0);
        double4 acc[VPL];
#pragma unroll
        for (int v = 0; v < VPL; v++) {
            acc[v] = make_double4(0.0, 0.0, 0.0, 0.0);
            const int c = lane + 32 * v;
            if (c < D4)
                for (int r = r0; r <= r1; r++) {
                    const float4 x = sg[(size_t)r * D4 + c];
                    acc[v].x += (double)x.x; acc[v].y += (double)x.y;
                    acc[v].z += (double)x.z; acc[v].w += (double)x.w;
                }
        }
        if (wh) {  // the whole row is in this tile
#pragma unroll
            for (int v = 0; v < VPL; v++) {
                const int c = lane + 32 * v;
                if (c < D4)
                    st[(size_t)s * D4 + c] = SR::nar(
                        sgd(SR::wid(sw[(size_t)wr * D4 + c]), Acc4{acc[v].x, acc[v].y, acc[v].z, acc[v].w}, A.lr));
            }
        } else {
            // 3. a piece of a row spanning tiles [kf, kl]: slot 0 of tile k
            // if the row holds the tile's first occurrence, else slot 1
            // (only possible in the row's first tile)
            const uint32_t u = __shfl_sync(0xffffffffu, uid, r0);
            // a piece is the tile's head row (r0 = 0) or its tail row (r1 = the last row)
            const int src = r0 == 0 ? 0 : r1;
            uint32_t slo = __shfl_sync(0xffffffffu, eslo, src), shi = __shfl_sync(0xffffffffu, eshi, src);
            if (slo == EMPTY) {
                if (lane == 0) {
                    slo = __ldg(A.bb.seg_off + (size_t)t * g.n1 + u);
                    shi = __ldg(A.bb.seg_off + (size_t)t * g.n1 + u + 1);
                }
                slo = __shfl_sync(0xffffffffu, slo, 0);
                shi = __shfl_sync(0xffffffffu, shi, 0);
            }
            const int kf = (int)(slo / (uint32_t)TR), kl = (int)((shi - 1u) / (uint32_t)TR);
            const int npc = kl - kf + 1;
            auto pslot = [&](int kk) { return (kk == kf && slo != (uint32_t)(kf * TR)) ? 1 : 0; };
            auto piece = [&](int kk) { return A.tpart + (((size_t)t * NT + kk) * 2 + pslot(kk)) * g.D; };
            double *mine = piece(k);
#pragma unroll
            for (int v = 0; v < VPL; v++) {
                const int c = lane + 32 * v;
                if (c < D4) reinterpret_cast<double4 *>(mine)[c] = acc[v];
            }
            if (A.tp2) continue;  // two-phase: k_bwd_rows folds the pieces
            bool go = true;
            int step = 1, cnt = npc;
            if (npc > 8) {  // level 1: groups of 8 consecutive pieces
                const int gi = (k - kf) / 8, g0 = kf + 8 * gi, gsz = min(8, kl - g0 + 1);
                uint32_t *gc = A.grp_cnt + ((size_t)t * NT + g0) * 2 + pslot(g0);
                go = warp_arrive_last(gc, (uint32_t)gsz, (A.diag & 256) != 0);
                if (go) {
                    if (lane == 0) *gc = 0u;
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        const int c = lane + 32 * v;
                        if (c >= D4) continue;
                        double4 m = make_double4(0.0, 0.0, 0.0, 0.0);
                        for (int q0 = 0; q0 < gsz; q0 += 4) {
                            double4 x[4];
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (q0 + q < gsz) x[q] = ld_piece(piece(g0 + q0 + q) + 4 * c);
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (q0 + q < gsz) dadd4(m, x[q]);
                        }
                        reinterpret_cast<double4 *>(piece(g0))[c] = m;
                    }
                }
                step = 8;
                cnt = (npc + 7) / 8;
            }
            if (go) {
                uint32_t *rc = A.seg_cnt + tb + u;
                if (warp_arrive_last(rc, (uint32_t)cnt, (A.diag & 256) != 0)) {
                    if (lane == 0) *rc = 0u;
#pragma unroll
                    for (int v = 0; v < VPL; v++) {
                        const int c = lane + 32 * v;
                        if (c >= D4) continue;
                        double4 m = make_double4(0.0, 0.0, 0.0, 0.0);
                        for (int q0 = 0; q0 < cnt; q0 += 4) {
                            double4 x[4];
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (q0 + q < cnt) x[q] = ld_piece(piece(kf + (q0 + q) * step) + 4 * c);
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (q0 + q < cnt) dadd4(m, x[q]);
                        }
                        typename SR::V *wp = st + (size_t)s * D4 + c;
                        *wp = SR::nar(sgd(SR::wid(*wp), Acc4{m.x, m.y, m.z, m.w}, A.lr));
                    }
                }
            }
        }
    }
}

#ifndef SP_META2
#define SP_META2 1  // k_bwd_tile: metadata two tiles ahead (0: one tile ahead, A/B)
#endif
#ifndef SP_BWD_TILE_MINB
#define SP_BWD_TILE_MINB 12  // resident warps per SM the registers are sized for (<= 152 regs; 16 KB of staging per warp at D = 128 fits 13-14 per SM anyway)
#endif
template <int VPL, bool BF = false>
__global__ void __launch_bounds__(32, VPL >= 2 ? SP_BWD_TILE_MINB / 2 : SP_BWD_TILE_MINB)
    k_bwd_tile(TrainArgs A, const __grid_constant__ CUtensorMap tmg, const __grid_constant__ CUtensorMap tms) {
    using SR = SRow<BF>;  // fp32 or bf16 Storage rows (R28)
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    const bool dead = *A.err != NO_ERR;  // (no work, but still counted out: the tile counters reset)
    const Geometry g = A.g;
    const int D4 = g.D / 4, TR = A.tr, NT = A.ntiles;
    const uint32_t rowb = (uint32_t)g.D * 4u, rowsb = (uint32_t)D4 * SR::bytes;  // gradient / Storage row bytes
    const int lane = threadIdx.x;
    float4 *sg = reinterpret_cast<float4 *>(sm);  // [TR][D4] gradient rows of the tile
    typename SR::V *sw = reinterpret_cast<typename SR::V *>(sg + (size_t)TR * D4);  // [TR][D4] Storage rows
    const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
    typename SR::V *st = reinterpret_cast<typename SR::V *>(A.storage);
    if (lane == 0) bar_init(&bar);
    __syncwarp();
    // a tile's metadata, one load wave: lane r holds sorted occurrence r, its
    // unique and its Storage slot (frozen at Plan); lane 0 also the unique
    // before the tile, lane nrows-1 the one after it (does a row cross the
    // tile's edges?)
    struct Meta { uint32_t occ, uid, slot, prev, next, slo, shi; };
    const uint32_t L = (uint32_t)g.L;
    auto bagof = [&](uint32_t occ) { return L == 1u ? occ : occ / L; };  // (no division for L = 1)
    const int total = dead ? 0 : g.T * NT;  // (< 2^31: T < 2^16 tables, NT <= n)
    auto load_meta = [&](int tile, Meta &m) {
        m = Meta{0u, EMPTY, 0u, EMPTY, EMPTY, EMPTY, EMPTY};
        if (tile >= total) return;
        const int t = tile / NT, k = tile - t * NT;
        const int lo = k * TR, nrows = min(TR, g.n - lo);
        const size_t base = (size_t)t * g.n + lo;
        if (lane < nrows) {
            m.occ = __ldg(A.bb.sorted_occ + base + lane);
            m.uid = __ldg(A.bb.sorted_uid + base + lane);  // EMPTY: padding (sorts last)
            m.slot = __ldg(A.bb.sorted_slot + base + lane);
        }
        if (lane == 0 && lo > 0) m.prev = __ldg(A.bb.sorted_uid + base - 1);
        if (lane == nrows - 1 && lo + nrows < g.n) m.next = __ldg(A.bb.sorted_uid + base + nrows);
        // the edge rows' segment offsets (a row crossing the tile's edge is a piece)
        if ((lane == 0 || lane == nrows - 1) && m.uid != EMPTY) {
            m.slo = __ldg(A.bb.seg_off + (size_t)t * g.n1 + m.uid);
            m.shi = __ldg(A.bb.seg_off + (size_t)t * g.n1 + m.uid + 1);
        }
    };
    // metadata two tiles ahead: `cur` for this tile, `nxt` for T(i+1) (loaded
    // during tile i-1), `nxt2` for T(i+2) (loaded during tile i), so both
    // levels of the load chain (uid -> segment offsets) hide behind a tile
    Meta cur, nxt, nxt2;
    load_meta(blockIdx.x, cur);  // (Plan's output: complete before the forward ran)
#if SP_META2
    load_meta(blockIdx.x + (int)gridDim.x, nxt);
#define SP_LOAD_NEXT_META() load_meta(after2, nxt2)
#else  // (A/B) one tile ahead
#define SP_LOAD_NEXT_META() load_meta(after, nxt)
#endif
    griddep_wait();  // (PDL) the surrogate's gradients are complete from here on
    unsigned long long *spn = span_base(A.span, SPK_BWD, A.span_b);
    span_mark(spn, 0);
    uint32_t parity = 0;
    // tile order: blockIdx.x, + G, + 2G, then claimed (3G + claim) when
    // A.tctr is set, else + 3G, + 4G, ... (static).  A claim is issued two
    // tiles before its index is needed (its latency hides behind two tiles).
    // Claims are spread over TCTR_GROUPS counters (one 128-B line each; one
    // same-address counter serialised ~7k claims at the L2): CTA c claims
    // from group j = c % TCTR_GROUPS, whose i-th claim is tile 3G + j + i*TCTR_GROUPS
    uint32_t *ctrs = A.tctr ? A.tctr + (size_t)(A.span_b % RING) * TCTR_STRIDE : nullptr;
    const int grp = (int)(blockIdx.x % TCTR_GROUPS);
    uint32_t *ctr = ctrs ? ctrs + grp * 32 : nullptr;
    const int G = (int)gridDim.x;
    int after = min(total, (int)blockIdx.x + G);       // T(i+1): its metadata loads during tile T(i)
    int after2 = min(total, (int)blockIdx.x + 2 * G);  // T(i+2)
    // pending claim (lane 0) for T(i+3), issued one tile earlier.  Indices
    // only grow along a CTA's sequence (static ones < 3G <= claimed ones, a
    // counter only grows), so once one is >= total all later ones are: no
    // claimed tile below total is ever dropped.
    uint32_t pend = 0;
    if (ctr && lane == 0) pend = atomicAdd(ctr, 1u);
    for (int tile = blockIdx.x; tile < total;) {
        const Meta m = cur;
        // claim T(i+4) now; its index is needed two tiles from here
        uint32_t claim = 0;
        if (ctr && lane == 0 && after2 < total) claim = atomicAdd(ctr, 1u);
        auto advance = [&]() {
            cur = nxt;
#if SP_META2
            nxt = nxt2;
#endif
            tile = after;
            after = after2;
            if (after2 < total)
                after2 = ctr ? min(total, 3 * G + grp + TCTR_GROUPS * (int)__shfl_sync(0xffffffffu, pend, 0))
                             : min(total, after2 + G);
            pend = claim;
        };
        const int t = tile / NT, k = tile - t * NT;
        const int lo = k * TR;
        const int nrows = min(TR, g.n - lo);
        const uint32_t uid = m.uid, slot = m.slot;
        const bool act = uid != EMPTY;
        const unsigned amask = __ballot_sync(0xffffffffu, act);
        if (amask == 0u) {  // (warp-uniform) all padding
            SP_LOAD_NEXT_META();
            advance();
            continue;
        }
        const int nact = 32 - __clz(amask);  // active rows are a prefix
        const uint32_t up = __shfl_up_sync(0xffffffffu, uid, 1), dn = __shfl_down_sync(0xffffffffu, uid, 1);
        const uint32_t prevu = lane == 0 ? m.prev : up;
        const uint32_t nextu = lane == nrows - 1 ? m.next : dn;  // (padding: EMPTY)
        const bool first = act && prevu != uid;
        const bool lastr = act && (lane == nact - 1 || nextu != uid);  // (a segment ends at the tile's edge)
        const uint32_t uid_last = __shfl_sync(0xffffffffu, uid, nact - 1);
        const bool tail_open = __shfl_sync(0xffffffffu, nextu == uid, nact - 1);
        const bool whole = first && !(uid == uid_last && tail_open);  // (lane 0 of an open head is not `first`)
        const unsigned wmask = __ballot_sync(0xffffffffu, whole);
        const unsigned lmask = __ballot_sync(0xffffffffu, lastr);
        if (A.diag & 128) {  // timing diagnostic: no staging (the fold reads stale shared memory)
            SP_LOAD_NEXT_META();
        } else if (A.g4) {
            // TMA tile::gather4: lane q fetches tile rows 4q..4q+3 (the last
            // group padded with the last row) and lane q the Storage rows of
            // whole segments 4q..4q+3 (compacted: the k-th whole segment's row
            // at sw[k]); one request per 4 rows
            const int ng = (nact + 3) >> 2, nw = __popc(wmask), nsg = (nw + 3) >> 2;
            if (lane == 0) bar_expect(&bar, (uint32_t)(4 * ng) * rowb + (uint32_t)(4 * nsg) * rowsb);
            __syncwarp();
            const uint32_t grow = (uint32_t)t * (uint32_t)g.N + bagof(m.occ);
            uint32_t gr[4], sr[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                gr[i] = __shfl_sync(0xffffffffu, grow, min(4 * lane + i, nact - 1));
                const int j = min(4 * lane + i, max(nw - 1, 0));
                const int pos = nw ? (int)__fns(wmask, 0, j + 1) : 0;
                sr[i] = __shfl_sync(0xffffffffu, slot, pos & 31);
            }
            if (lane < ng) rows4_g2s(sg + (size_t)4 * lane * D4, &tmg, gr[0], gr[1], gr[2], gr[3], &bar);
            if (lane < nsg) rows4_g2s(sw + (size_t)4 * lane * D4, &tms, sr[0], sr[1], sr[2], sr[3], &bar);
            SP_LOAD_NEXT_META();
            while (!bar_try(&bar, parity)) {
            }
            parity ^= 1u;
        } else if (A.bwd_tma) {  // one TMA bulk copy per row, completion on the mbarrier
            if (lane == 0) bar_expect(&bar, (uint32_t)__popc(amask) * rowb + (uint32_t)__popc(wmask) * rowsb);
            __syncwarp();
            if (act) row_g2s(sg + (size_t)lane * D4, grad + ((size_t)t * g.N + bagof(m.occ)) * D4, rowb, &bar);
            if (whole) row_g2s(sw + (size_t)lane * D4, st + (size_t)slot * D4, rowsb, &bar);
            SP_LOAD_NEXT_META();  // the next tile's metadata, in flight with the copies
            while (!bar_try(&bar, parity)) {
            }
            parity ^= 1u;
        } else {
            // (A/B) 16-B async copies (LDGSTS), one warp-wide instruction per
            // 512 B of row: measured slower than the bulk copies (TB pipelined
            // 54 vs 38 us in-situ span; profiles/r02_xs3_sweep.txt)
            for (int r = 0; r < nact; r++) {
                const uint32_t o = __shfl_sync(0xffffffffu, m.occ, r);
                const float4 *src = grad + ((size_t)t * g.N + o / (uint32_t)g.L) * D4;
                for (int c = lane; c < D4; c += 32) cp16(sg + (size_t)r * D4 + c, src + c);
            }
            for (unsigned wm = wmask; wm; wm &= wm - 1) {
                const int r = __ffs(wm) - 1;
                const uint32_t sl = __shfl_sync(0xffffffffu, slot, r);
                const char *src = reinterpret_cast<const char *>(st + (size_t)sl * D4);
                char *dst = reinterpret_cast<char *>(sw + (size_t)r * D4);
                for (uint32_t c = lane; c < rowsb / 16u; c += 32) cp16(dst + 16 * c, src + 16 * c);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            SP_LOAD_NEXT_META();  // the next tile's metadata, in flight with the copies
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
        }
        if (!(A.diag & 64)) bwd_fold_tile<VPL, BF>(A, t, k, lmask, wmask, slot, uid, sg, sw, m.slo, m.shi);  // (64: no fold, timing)
        // the tile's shared rows are consumed (generic proxy) before the next
        // tile's bulk copies (async proxy) overwrite them
        __syncwarp();
        if (A.bwd_tma || A.g4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        advance();
    }
    span_mark(spn, 1);
#undef SP_LOAD_NEXT_META
    if (ctrs && lane == 0) {  // every claim of every CTA precedes its exit: the last one out resets
        if (atomicAdd(ctrs + TCTR_GROUPS * 32, 1u) == gridDim.x - 1) {
            for (int j = 0; j <= TCTR_GROUPS; j++) ctrs[j * 32] = 0u;
        }
    }
}

// Second phase of the two-phase backward: every row spanning tiles [kf, kl]
// left one fp64 piece per tile (k_bwd_tile); here the pieces are folded and
// SGD applied.  The owner of such a row is its first tile kf (the row starts
// inside it and runs past its end).  A CTA takes 32 tiles at a time: warp 0
// checks them (one lane per tile, one load wave) and lists the owners in
// shared memory; a row of <= BWD2_SMALL pieces is then folded by one warp,
// in tile order (8 pieces in flight per round); a longer one (the Zipf
// head: up to n/TR pieces) by all 8 warps -- warp w sums pieces kf+w, kf+w+8,
// ... in order, then warp 0 adds the 8 partials in warp order.  The fold
// shape depends only on the batch.
constexpr int BWD2_SMALL = 16;  // (8 / 16 / 32 measured equal: profiles/r02_s3_ab.txt)
template <int VPL, bool BF>
__global__ void __launch_bounds__(256, 2) k_bwd_rows(TrainArgs A) {
    using SR = SRow<BF>;
    extern __shared__ __align__(16) unsigned char sm2[];
    double4 *spart = reinterpret_cast<double4 *>(sm2);  // [8][D4] partials of a long row
    __shared__ uint4 s_item[32];                         // (t, u, kf, kl) of each owner found
    __shared__ uint32_t s_slo[32], s_slot[32];
    __shared__ uint32_t s_small, s_big;                  // ballots of short / long owners
    const bool dead = *A.err != NO_ERR;
    const Geometry g = A.g;
    const int D4 = g.D / 4, TR = A.tr, NT = A.ntiles;
    const int total = dead ? 0 : g.T * NT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    typename SR::V *st = reinterpret_cast<typename SR::V *>(A.storage);
    unsigned long long *spn = span_base(A.span, SPK_BWD, A.span_b);
    span_mark(spn, 0, SPAN_BWD2_OFF);
    auto piece = [&](int t, int kk, int kf, uint32_t slo) {
        const int ps = (kk == kf && slo != (uint32_t)(kf * TR)) ? 1 : 0;
        return reinterpret_cast<const double4 *>(A.tpart + (((size_t)t * NT + kk) * 2 + ps) * g.D);
    };
    auto apply = [&](uint32_t slot, int c, const double4 &m) {
        typename SR::V *wp = st + (size_t)slot * D4 + c;
        *wp = SR::nar(sgd(SR::wid(*wp), Acc4{m.x, m.y, m.z, m.w}, A.lr));
    };
    bool waited = false;
    for (int base = blockIdx.x * 32; base < total; base += gridDim.x * 32) {
        // 1. owners among tiles base..base+31 (Plan's output: readable before the wait)
        if (warp == 0) {
            const int tile = base + lane;
            uint4 it = make_uint4(EMPTY, 0u, 0u, 0u);
            uint32_t slo = 0, slot = 0;
            if (tile < total) {
                const int t = tile / NT, k = tile - t * NT;
                const int lo = k * TR, nrows = min(TR, g.n - lo);
                if (lo + nrows < g.n) {
                    const size_t tb = (size_t)t * g.n;
                    // one wave: the tail row, the row after it and the tail row's
                    // slot (every occurrence of a row has the same slot); then its
                    // segment offsets
                    const uint32_t u = __ldg(A.bb.sorted_uid + tb + lo + nrows - 1);
                    const uint32_t un = __ldg(A.bb.sorted_uid + tb + lo + nrows);
                    const uint32_t sl = __ldg(A.bb.sorted_slot + tb + lo + nrows - 1);
                    if (u != EMPTY && u == un) {
                        slo = __ldg(A.bb.seg_off + (size_t)t * g.n1 + u);
                        const uint32_t shi = __ldg(A.bb.seg_off + (size_t)t * g.n1 + u + 1);
                        if (slo >= (uint32_t)lo) {
                            slot = sl;
                            it = make_uint4((uint32_t)t, u, (uint32_t)k, (shi - 1u) / (uint32_t)TR);
                        }
                    }
                }
            }
            const bool own = it.x != EMPTY;
            const bool big = own && (int)(it.w - it.z) + 1 > (A.bwd2_small > 0 ? A.bwd2_small : BWD2_SMALL);
            s_item[lane] = it;
            s_slo[lane] = slo;
            s_slot[lane] = slot;
            const unsigned bs = __ballot_sync(0xffffffffu, own && !big), bb = __ballot_sync(0xffffffffu, big);
            if (lane == 0) { s_small = bs; s_big = bb; }
        }
        __syncthreads();
        const unsigned small = s_small, bigm = s_big;
        if (!(small | bigm)) continue;  // (CTA-uniform; the next chunk's writes follow this barrier)
        if (!waited) {  // (PDL) the pieces of k_bwd_tile are complete from here on
            griddep_wait();
            waited = true;
        }
        // 2. short rows: owner i of the chunk goes to warp (rank of i) % 8
        {
            unsigned m = small;
            for (int r = 0; m; r++, m &= m - 1) {
                if ((r & 7) != warp) continue;
                const int i = __ffs(m) - 1;
                const uint4 it = s_item[i];
                const int t = (int)it.x, kf = (int)it.z, npc = (int)(it.w - it.z) + 1;
                const uint32_t slo = s_slo[i], slot = s_slot[i];
#pragma unroll 1
                for (int v = 0; v < VPL; v++) {
                    const int c = lane + 32 * v;
                    if (c >= D4) continue;
                    // (2 <= npc <= the threshold) 8 pieces in flight per round, added in tile order
                    double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
                    for (int q0 = 0; q0 < npc; q0 += 8) {
                        double4 x[8];
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            if (q0 + q < npc) x[q] = ldcg_d4(piece(t, kf + q0 + q, kf, slo) + c);
                        if (q0 == 0) acc = x[0];
                        else dadd4(acc, x[0]);
#pragma unroll
                        for (int q = 1; q < 8; q++)
                            if (q0 + q < npc) dadd4(acc, x[q]);
                    }
                    apply(slot, c, acc);
                }
            }
        }
        // 3. long rows: all 8 warps, then warp 0 in warp order
        for (unsigned m = bigm; m; m &= m - 1) {
            const int i = __ffs(m) - 1;
            const uint4 it = s_item[i];
            const int t = (int)it.x, kf = (int)it.z, np = (int)(it.w - it.z) + 1;
            const uint32_t slo = s_slo[i];
#pragma unroll 1
            for (int v = 0; v < VPL; v++) {
                const int c = lane + 32 * v;
                if (c >= D4) continue;
                double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
                for (int q0 = warp; q0 < np; q0 += 32) {  // pieces q0, q0+8, q0+16, q0+24 in flight
                    double4 x0, x1, x2, x3;
                    x0 = ldcg_d4(piece(t, kf + q0, kf, slo) + c);
                    if (q0 + 8 < np) x1 = ldcg_d4(piece(t, kf + q0 + 8, kf, slo) + c);
                    if (q0 + 16 < np) x2 = ldcg_d4(piece(t, kf + q0 + 16, kf, slo) + c);
                    if (q0 + 24 < np) x3 = ldcg_d4(piece(t, kf + q0 + 24, kf, slo) + c);
                    dadd4(acc, x0);
                    if (q0 + 8 < np) dadd4(acc, x1);
                    if (q0 + 16 < np) dadd4(acc, x2);
                    if (q0 + 24 < np) dadd4(acc, x3);
                }
                spart[(size_t)warp * D4 + c] = acc;
            }
            __syncthreads();
            if (warp == 0) {
#pragma unroll
                for (int v = 0; v < VPL; v++) {
                    const int c = lane + 32 * v;
                    if (c >= D4) continue;
                    double4 acc = spart[c];
                    for (int ww = 1; ww < 8; ww++) dadd4(acc, spart[(size_t)ww * D4 + c]);
                    apply(s_slot[i], c, acc);
                }
            }
            __syncthreads();
        }
        __syncthreads();  // s_item is rewritten by the next chunk
    }
    span_mark(spn, 1, SPAN_BWD2_OFF);
}

// Warp-specialised variant (A/B, SP_BWD_WS=1): a CTA of two warps and two staging
// buffers.  Warp 0 (producer) reads a tile's metadata, derives the segment
// masks, hands them over in shared memory and issues the TMA copies of the
// tile's rows into a free buffer (mbarrier `full`, with the byte count);
// warp 1 (consumer) folds the previous buffer and releases it (mbarrier
// `empty`).  The copies of tile i+1 and the per-tile bookkeeping run while
// tile i is folded.  Same tiles, same fold (bwd_fold_tile), same results as
// k_bwd_tile.
template <int VPL>
__global__ void __launch_bounds__(64, VPL >= 2 ? 4 : 8)
    k_bwd_ws(TrainArgs A, const __grid_constant__ CUtensorMap tmg, const __grid_constant__ CUtensorMap tms) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[2], empty[2];
    __shared__ uint32_t s_slot[2][32], s_uid[2][32], s_lm[2], s_wm[2];
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4, TR = A.tr, NT = A.ntiles;
    const uint32_t rowb = (uint32_t)g.D * 4u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4 *stage0 = reinterpret_cast<float4 *>(sm);
    auto gbuf = [&](int b) { return stage0 + (size_t)b * 2 * TR * D4; };  // [TR][D4] gradient rows
    auto wbuf = [&](int b) { return gbuf(b) + (size_t)TR * D4; };         // [TR][D4] Storage rows
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[b])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&empty[b])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long total = (long long)g.T * NT;
    unsigned long long *spn = span_base(A.span, SPK_BWD, A.span_b);
    if (warp == 0) {
        // ---------------- producer
        const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
        const float4 *st = reinterpret_cast<const float4 *>(A.storage);
        uint32_t occ = 0, uid = EMPTY, slot = 0, prev = EMPTY, next = EMPTY;
        auto load_meta = [&](long long tile) {
            occ = 0; uid = EMPTY; slot = 0; prev = EMPTY; next = EMPTY;
            if (tile >= total) return;
            const int t = (int)(tile / NT), k = (int)(tile % NT);
            const int lo = k * TR, nrows = min(TR, g.n - lo);
            const size_t base = (size_t)t * g.n + lo;
            if (lane < nrows) {
                occ = __ldg(A.bb.sorted_occ + base + lane);
                uid = __ldg(A.bb.sorted_uid + base + lane);
                slot = __ldg(A.bb.sorted_slot + base + lane);
            }
            if (lane == 0 && lo > 0) prev = __ldg(A.bb.sorted_uid + base - 1);
            if (lane == nrows - 1 && lo + nrows < g.n) next = __ldg(A.bb.sorted_uid + base + nrows);
        };
        load_meta(blockIdx.x);
        griddep_wait();  // (PDL) the surrogate's gradients are complete from here on
        span_mark(spn, 0);
        uint32_t i = 0;
        for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, i++) {
            const int b = (int)(i & 1u);
            const uint32_t ph = (i >> 1) & 1u;
            const uint32_t m_occ = occ, m_uid = uid, m_slot = slot, m_prev = prev, m_next = next;
            const int t = (int)(tile / NT), k = (int)(tile % NT);
            const int nrows = min(TR, g.n - k * TR);
            const bool act = m_uid != EMPTY;
            const unsigned amask = __ballot_sync(0xffffffffu, act);
            unsigned lmask = 0u, wmask = 0u;
            int nact = 0;
            if (amask) {
                nact = 32 - __clz(amask);
                const uint32_t up = __shfl_up_sync(0xffffffffu, m_uid, 1), dn = __shfl_down_sync(0xffffffffu, m_uid, 1);
                const uint32_t prevu = lane == 0 ? m_prev : up;
                const uint32_t nextu = lane == nrows - 1 ? m_next : dn;
                const bool first = act && prevu != m_uid;
                const bool lastr = act && (lane == nact - 1 || nextu != m_uid);
                const uint32_t uid_last = __shfl_sync(0xffffffffu, m_uid, nact - 1);
                const bool tail_open = __shfl_sync(0xffffffffu, nextu == m_uid, nact - 1);
                const bool whole = first && !(m_uid == uid_last && tail_open);
                wmask = __ballot_sync(0xffffffffu, whole);
                lmask = __ballot_sync(0xffffffffu, lastr);
            }
            // the consumer has released buffer b (its use two tiles ago)
            while (!bar_try(&empty[b], ph ^ 1u)) {
            }
            s_slot[b][lane] = m_slot;
            s_uid[b][lane] = m_uid;
            if (lane == 0) {
                s_lm[b] = lmask;
                s_wm[b] = wmask;
            }
            __syncwarp();
            float4 *sg = gbuf(b), *sw = wbuf(b);
            if (A.g4 && amask) {
                const int ng = (nact + 3) >> 2, nw = __popc(wmask), nsg = (nw + 3) >> 2;
                if (lane == 0) bar_expect(&full[b], (uint32_t)(4 * ng + 4 * nsg) * rowb);
                __syncwarp();
                const uint32_t grow = (uint32_t)t * (uint32_t)g.N + m_occ / (uint32_t)g.L;
                uint32_t gr[4], sr[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    gr[q] = __shfl_sync(0xffffffffu, grow, min(4 * lane + q, nact - 1));
                    const int j = min(4 * lane + q, max(nw - 1, 0));
                    const int pos = nw ? (int)__fns(wmask, 0, j + 1) : 0;
                    sr[q] = __shfl_sync(0xffffffffu, m_slot, pos & 31);
                }
                if (lane < ng) rows4_g2s(sg + (size_t)4 * lane * D4, &tmg, gr[0], gr[1], gr[2], gr[3], &full[b]);
                if (lane < nsg) rows4_g2s(sw + (size_t)4 * lane * D4, &tms, sr[0], sr[1], sr[2], sr[3], &full[b]);
            } else {
                if (lane == 0) bar_expect(&full[b], (uint32_t)(__popc(amask) + __popc(wmask)) * rowb);
                __syncwarp();
                if (act) row_g2s(sg + (size_t)lane * D4, grad + ((size_t)t * g.N + m_occ / (uint32_t)g.L) * D4, rowb, &full[b]);
                if ((wmask >> lane) & 1u) row_g2s(sw + (size_t)lane * D4, st + (size_t)m_slot * D4, rowb, &full[b]);
            }
            load_meta(tile + gridDim.x);
        }
    } else {
        // ---------------- consumer
        griddep_wait();
        uint32_t i = 0;
        for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, i++) {
            const int b = (int)(i & 1u);
            const uint32_t ph = (i >> 1) & 1u;
            while (!bar_try(&full[b], ph)) {
            }
            const unsigned lmask = s_lm[b], wmask = s_wm[b];
            const uint32_t slot = s_slot[b][lane], uid = s_uid[b][lane];
            const int t = (int)(tile / NT), k = (int)(tile % NT);
            if (lmask) bwd_fold_tile<VPL>(A, t, k, lmask, wmask, slot, uid, gbuf(b), wbuf(b));
            // buffer b consumed (generic proxy) before the producer's next
            // copies (async proxy) into it
            __syncwarp();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[b])) : "memory");
        }
    }
    __syncthreads();
    span_mark(spn, 1);
}

// generic D (D/4 not a power-of-two multiple of 32): one warp per row,
// strided columns; hot rows and chunk records both folded in ascending
// occurrence order by that warp (sequential fp64 fold)
__global__ void __launch_bounds__(256) k_bwd_generic(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    const int wpb = blockDim.x / 32;
    const long long w0 = (long long)blockIdx.x * wpb + threadIdx.x / 32, ws = (long long)gridDim.x * wpb;
    for (int t = 0; t < g.T; t++) {
        const float4 *gb = grad + (size_t)t * g.N * D4;
        const uint32_t nhot = A.bb.nhot[t];
        for (long long h = w0; h < nhot; h += ws) {
            const uint4 hr = A.bb.hot_rec[(size_t)t * g.nh + h];
            if (hr.w != 0) continue;  // segment 0 owns the whole row
            const uint32_t nseg = hr.z >> HOT_LEN_BITS;
            uint32_t len = 0;
            for (uint32_t k = 0; k < nseg; k++) len += A.bb.hot_rec[(size_t)t * g.nh + h + k].z & HOT_LEN_MASK;
            const uint32_t *occ = A.bb.sorted_occ + (size_t)t * g.n + hr.y;
            for (int col = lane; col < D4; col += 32) {
                Acc4 a{0.0, 0.0, 0.0, 0.0};
                for (uint32_t i = 0; i < len; i++) acc_add(a, gb[(size_t)(occ[i] / (uint32_t)g.L) * D4 + col]);
                st[(size_t)hr.x * D4 + col] = sgd(st[(size_t)hr.x * D4 + col], a, A.lr);
            }
        }
        const uint32_t total = A.bb.nchunks[t];
        for (long long c = w0; c < total; c += ws) {
            const ChunkRec &rc = A.bb.chunk_rec[(size_t)t * g.nc + c];
            const uint32_t slot = rc.slot, len = rc.meta;
            for (int col = lane; col < D4; col += 32) {
                Acc4 a{0.0, 0.0, 0.0, 0.0};
                for (uint32_t i = 0; i < len; i++) acc_add(a, gb[(size_t)rc.bag[i] * D4 + col]);
                st[(size_t)slot * D4 + col] = sgd(st[(size_t)slot * D4 + col], a, A.lr);
            }
        }
    }
}

// -------------------------------------------------------------- surrogate
// Streaming: each thread keeps SU float4 loads in flight (loads first, then
// the fmas and stores), so latency, not occupancy, is covered; element i's
// result does not depend on the grid.
constexpr int SU = 4;
__global__ void __launch_bounds__(256) k_surrogate(const float4 *p, float4 *g, long long n4,
                                                   float gamma, float delta, unsigned long long *span) {
    griddep_wait();  // (PDL) pooled is complete from here on
    span_mark(span, 0);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += SU * stride) {
        float4 x[SU];
#pragma unroll
        for (int u = 0; u < SU; u++) {
            const long long i = i0 + u * stride;
            if (i < n4) x[u] = __ldcs(p + i);
        }
#pragma unroll
        for (int u = 0; u < SU; u++) {
            const long long i = i0 + u * stride;
            if (i < n4) {
                float4 y;
                y.x = fmaf(gamma, x[u].x, delta);
                y.y = fmaf(gamma, x[u].y, delta);
                y.z = fmaf(gamma, x[u].z, delta);
                y.w = fmaf(gamma, x[u].w, delta);
                g[i] = y;
            }
        }
    }
    if (span) {
        __syncthreads();
        span_mark(span, 1);
    }
}

// --------------------------------------------------------------- launchers
// Per-device caches: a process may hold contexts on several GPUs, and kernel
// attributes / occupancy are per device.
static std::mutex g_dev_mu;

int device_sms() {
    static int sms[256] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (dev < 0 || dev >= 256) return 148;
    if (!sms[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = n > 0 ? n : 148;
    }
    return sms[dev];
}

// resident CTAs of a kernel on the whole GPU (a persistent grid never waits
// for a second wave of a latency-bound kernel); the carveout hint is applied
// on first use on each device
template <typename K>
static int resident_ctas(K kernel, int threads) {
    static std::map<std::pair<const void *, int>, int> caps;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        auto it = caps.find({reinterpret_cast<const void *>(kernel), dev});
        if (it != caps.end()) return it->second;
    }
    apply_carveout(kernel);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int cap = per_sm * device_sms();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    caps[{reinterpret_cast<const void *>(kernel), dev}] = cap;
    return cap;
}

template <typename K, typename... Args>
static void launch_maybe_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t s, bool pdl, Args... args) {
    if (pdl && g_pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kernel, args...);
    } else {
        kernel<<<grid, block, smem, s>>>(args...);
    }
}

template <int G, int VPL, typename K>
static void launch_sized(K kernel, long long groups, const TrainArgs &a, cudaStream_t s, bool pdl = false) {
    const int cap = resident_ctas(kernel, 256);  // per kernel instance and device
    long long blocks = (groups + (256 / G) - 1) / (256 / G);
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    launch_maybe_pdl(kernel, grid, 256, 0, s, pdl, a);
}

#define SP_DISPATCH_D(D4, KERNEL, GROUPS, ARGS, STREAM, PDL)                                   \
    switch (D4) {                                                                              \
        case 1: launch_sized<1, 1>(KERNEL<1, 1>, GROUPS, ARGS, STREAM, PDL); break;            \
        case 2: launch_sized<2, 1>(KERNEL<2, 1>, GROUPS, ARGS, STREAM, PDL); break;            \
        case 4: launch_sized<4, 1>(KERNEL<4, 1>, GROUPS, ARGS, STREAM, PDL); break;            \
        case 8: launch_sized<8, 1>(KERNEL<8, 1>, GROUPS, ARGS, STREAM, PDL); break;            \
        case 16: launch_sized<16, 1>(KERNEL<16, 1>, GROUPS, ARGS, STREAM, PDL); break;         \
        case 32: launch_sized<32, 1>(KERNEL<32, 1>, GROUPS, ARGS, STREAM, PDL); break;         \
        case 64: launch_sized<32, 2>(KERNEL<32, 2>, GROUPS, ARGS, STREAM, PDL); break;         \
        case 128: launch_sized<32, 4>(KERNEL<32, 4>, GROUPS, ARGS, STREAM, PDL); break;        \
        case 256: launch_sized<32, 8>(KERNEL<32, 8>, GROUPS, ARGS, STREAM, PDL); break;        \
        default: launch_sized<32, 1>(KERNEL##_generic, GROUPS, ARGS, STREAM, false); break;    \
    }

cudaError_t launch_forward(const TrainArgs &a, cudaStream_t s) {
    const int D4 = a.g.D / 4;
    if (a.g.bf16 && a.g.pad) {
        SP_DISPATCH_D(D4, k_fwd_pad_bf, (long long)a.g.T * a.g.N, a, s, false);
    } else if (a.g.bf16) {
        SP_DISPATCH_D(D4, k_fwd_bf, (long long)a.g.T * a.g.N, a, s, false);
    } else if (a.g.pad) {
        SP_DISPATCH_D(D4, k_fwd_pad, (long long)a.g.T * a.g.N, a, s, false);
    } else {
        SP_DISPATCH_D(D4, k_fwd, (long long)a.g.T * a.g.N, a, s, false);
    }
    return cudaGetLastError();
}

// occurrences per hot-row segment: one round of RB rows per lane group of
// the k_bwd instance that D dispatches to (generic D: 64).  (Half-width lane
// groups, two float4 per lane, were measured slower: 20.7 vs 16.4 us.)
// occurrences per hot-row segment (one warp of k_bwd folds a segment;
// generic D: one warp too).  SP_HOT_SEG overrides (A/B).
int backward_hot_segment(int D) {
    (void)D;
    int hs = 32;
    if (const char *e = getenv("SP_HOT_SEG")) hs = atoi(e) >= CH ? atoi(e) : hs;
    // (segment lengths are packed in HOT_LEN_BITS of the hot record)
    return hs < CH ? CH : (hs > HOT_SEG_MAX ? HOT_SEG_MAX : hs);
}

// k_bwd_tile: rows per tile so that a warp's two staging areas (gradient and
// Storage rows) take 16 KB (at most 32 rows: one per lane), i.e. 13 warps
// per SM.  SP_BWD_TR overrides (A/B).
int backward_tile_rows(int D) {
    int tr = 8192 / (D * 4);
    if (const char *e = getenv("SP_BWD_TR")) tr = atoi(e);
    return tr < 1 ? 1 : (tr > 32 ? 32 : tr);
}

bool backward_tiled() {
    const char *e = getenv("SP_BWD");
    return !(e && e[0] == 'r');
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda)
typedef CUresult (*tmap_encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static tmap_encode_fn tmap_encode() {
    static tmap_encode_fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<tmap_encode_fn>(p);
        (void)cudaGetLastError();
    });
    return fn;
}

// a [rows][D] fp32 matrix as a 2-D tensor map with a one-row box (the form
// tile::gather4 takes: tools/gather4_probe.cu)
static bool rows_map(CUtensorMap *m, const void *base, unsigned long long rows, int D, bool bf16 = false) {
    tmap_encode_fn enc = tmap_encode();
    if (!enc || !base || rows == 0 || D > 256 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    const int esz = bf16 ? 2 : 4;
    if ((D * esz) % 16) return false;  // row stride: a multiple of 16 B
    cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)rows}, gstr[1] = {(cuuint64_t)D * esz};
    cuuint32_t box[2] = {(cuuint32_t)D, 1}, es[2] = {1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
               const_cast<void *>(base), gdim, gstr, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_bwd_g4 = -1;  // SP_BWD_G4: 0 disables tile::gather4 (A/B)
static int g_bwd_ws = -1;  // SP_BWD_WS=1: the warp-specialised k_bwd_ws (A/B: measured slower, 52 vs 36 us isolated
                           // on Terabyte: 6 consumer warps per SM fold less than 13 one-warp CTAs)

template <int VPL, bool BF>
static void launch_bwd_tile(const TrainArgs &a0, cudaStream_t s) {
    TrainArgs a = a0;
    CUtensorMap tmg, tms;
    std::memset(&tmg, 0, sizeof tmg);
    std::memset(&tms, 0, sizeof tms);
    if (g_bwd_g4 < 0) {
        const char *e = getenv("SP_BWD_G4");
        g_bwd_g4 = e ? (atoi(e) != 0) : 1;
    }
    // a tensor copy's shared-memory destination must be 128-B aligned: a
    // group of 4 gradient rows (16*D bytes) is when D % 8 == 0, of 4 bf16
    // Storage rows (8*D bytes) when D % 16 == 0
    a.g4 = g_bwd_g4 && a.bwd_tma && a.tr % 4 == 0 && a.tr <= 32 && a.g.D % (BF ? 16 : 8) == 0 &&
           rows_map(&tmg, a.grad, (unsigned long long)a.g.T * a.g.N, a.g.D) &&
           rows_map(&tms, a.storage, (unsigned long long)a.srows, a.g.D, BF);
    const size_t smem = (size_t)a.tr * a.g.D * (sizeof(float) + (BF ? 2 : sizeof(float)));
    // (device, kernel) -> resident CTAs
    static std::map<std::pair<int, const void *>, int> caps;
    const void *kid = reinterpret_cast<const void *>(k_bwd_tile<VPL, BF>);
    int dev = 0;
    cudaGetDevice(&dev);
    int cap = 0;
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        auto it = caps.find({dev, kid});
        if (it != caps.end()) cap = it->second;
    }
    if (!cap) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_tile<VPL, BF>, 32, smem) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        cap = per_sm * device_sms();
        std::lock_guard<std::mutex> lk(g_dev_mu);
        caps[{dev, kid}] = cap;
    }
    const long long tiles = (long long)a.g.T * a.ntiles;
    if (g_bwd_ws < 0) {
        const char *e = getenv("SP_BWD_WS");
        g_bwd_ws = e ? (atoi(e) != 0) : 0;
    }
    if (!BF && g_bwd_ws && a.bwd_tma) {  // two warps, two staging buffers per CTA (fp32 Storage only)
        a.tp2 = 0;  // (one phase: last-arriver counters)
        const size_t smem2 = 2 * smem;
        static std::map<std::pair<int, size_t>, int> caps2;
        int cap2 = 0;
        {
            std::lock_guard<std::mutex> lk(g_dev_mu);
            auto it = caps2.find({dev, smem2});
            if (it != caps2.end()) cap2 = it->second;
        }
        if (!cap2) {
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_ws<VPL>, 64, smem2) != cudaSuccess ||
                per_sm < 1)
                per_sm = 1;
            cap2 = per_sm * device_sms();
            std::lock_guard<std::mutex> lk(g_dev_mu);
            caps2[{dev, smem2}] = cap2;
        }
        int grid2 = (int)(tiles < cap2 ? tiles : cap2);
        if (grid2 < 1) grid2 = 1;
        launch_maybe_pdl(k_bwd_ws<VPL>, grid2, 64, smem2, s, true, a, tmg, tms);
        return;
    }
    int grid = (int)(tiles < cap ? tiles : cap);
    if (grid < 1) grid = 1;
    launch_maybe_pdl(k_bwd_tile<VPL, BF>, grid, 32, smem, s, true, a, tmg, tms);
    if (a.tp2) {  // second phase: rows spanning tiles (32 tiles checked per CTA)
        long long g2 = (tiles + 31) / 32;
        if (g2 > SPAN_MAXCTA - SPAN_BWD2_OFF) g2 = SPAN_MAXCTA - SPAN_BWD2_OFF;
        if (g2 < 1) g2 = 1;
        launch_maybe_pdl(k_bwd_rows<VPL, BF>, (int)g2, 256, (size_t)64 * a.g.D, s, true, a);
    }
}

cudaError_t launch_backward(const TrainArgs &a, cudaStream_t s) {
    const int D4 = a.g.D / 4;
    if (a.tpart && a.g.bf16) {  // bf16 Storage: the tiled backward only
        if (D4 <= 32) launch_bwd_tile<1, true>(a, s);
        else if (D4 <= 64) launch_bwd_tile<2, true>(a, s);
        else if (D4 <= 128) launch_bwd_tile<4, true>(a, s);
        else launch_bwd_tile<8, true>(a, s);
        return cudaGetLastError();
    }
    if (a.tpart) {
        if (D4 <= 32) launch_bwd_tile<1, false>(a, s);
        else if (D4 <= 64) launch_bwd_tile<2, false>(a, s);
        else if (D4 <= 128) launch_bwd_tile<4, false>(a, s);
        else launch_bwd_tile<8, false>(a, s);
        return cudaGetLastError();
    }
    if (a.g.bf16) return cudaErrorInvalidValue;  // (the record-based k_bwd is fp32 only)
    // upper bound of work items: all chunks of all tables
    SP_DISPATCH_D(D4, k_bwd, (long long)a.g.T * a.g.nc, a, s, true);
    return cudaGetLastError();
}

cudaError_t launch_surrogate(const float *pooled, float *grad, long long count, float gamma,
                             float delta, cudaStream_t s, unsigned long long *span, long long span_b) {
    long long n4 = count / 4;
    long long blocks = (n4 + 256 * SU - 1) / (256 * SU);
    const long long cap = (long long)device_sms() * 8;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    launch_maybe_pdl(k_surrogate, grid, 256, 0, s, true, reinterpret_cast<const float4 *>(pooled),
                     reinterpret_cast<float4 *>(grad), n4, gamma, delta,
                     span ? span + (((size_t)SPK_SURR * RING + (size_t)(span_b % RING)) * SPAN_MAXCTA) * 2 : nullptr);
    return cudaGetLastError();
}

// attributes of the Train-stage kernels on the current device (sp_create)
cudaError_t configure_train_kernels() {
    apply_carveout(k_surrogate);
    // k_bwd_tile is sized by shared memory (one warp, up to 32 KB each): ask
    // for the largest carveout so that 6-7 CTAs fit per SM
    cudaFuncSetAttribute(k_bwd_tile<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<1, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<2, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<4, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_tile<8, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // k_bwd_rows: 8 fp64 partial rows of D (64 KB at D = 1024)
    cudaFuncSetAttribute(k_bwd_rows<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_rows<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_bwd_ws<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_ws<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_ws<4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_bwd_ws<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return cudaGetLastError();
}

}  // namespace sp
