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
//           occurrences (ascending occurrence order, contiguous in the sorted
//           occurrence list built at Plan) are summed in fp64 and the row is
//           updated in place, w = fmaf(-lr, (float)sum, w).  One owner per
//           unique row -> no atomics on Storage.  Long (hot, Zipf-skewed)
//           segments are split into chunks of CH occurrences whose fp64
//           partials are folded in chunk order by the last chunk to finish.
//   k_surrogate  the harness's MLP stand-in g = fmaf(gamma, pooled, delta).
#include "sp_internal.cuh"

#include <unordered_map>

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

__device__ __forceinline__ float4 ldg4(const float4 *p) { return __ldg(p); }

__device__ __forceinline__ void add4(float4 &a, const float4 &b) {
    a.x = a.x + b.x; a.y = a.y + b.y; a.z = a.z + b.z; a.w = a.w + b.w;
}

}  // namespace

// ---------------------------------------------------------------- forward
// G lanes per bag, VPL float4 per lane (D/4 = G*VPL).
template <int G, int VPL>
__global__ void __launch_bounds__(256) k_fwd(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const int L = A.g.L, D4 = A.g.D / 4;
    const long long nbags = (long long)A.g.T * A.g.N;
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    const float4 *st = reinterpret_cast<const float4 *>(A.storage);
    float4 *out = reinterpret_cast<float4 *>(A.pooled);
    for (long long bag = (long long)blockIdx.x * gpb + threadIdx.x / G; bag < nbags;
         bag += (long long)gridDim.x * gpb) {
        const uint32_t *so = A.bb.slot_of_occ + bag * L;
        float4 acc[VPL];
        {
            const uint32_t s = __ldg(so);
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[v] = ldg4(st + (size_t)s * D4 + lane + v * G);
        }
        int p = 1;
        for (; p + 4 <= L; p += 4) {  // 4 rows in flight, folded in p order
            uint32_t s[4];
#pragma unroll
            for (int q = 0; q < 4; q++) s[q] = __ldg(so + p + q);
            float4 r[4][VPL];
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int v = 0; v < VPL; v++) r[q][v] = ldg4(st + (size_t)s[q] * D4 + lane + v * G);
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int v = 0; v < VPL; v++) add4(acc[v], r[q][v]);
        }
        for (; p < L; p++) {
            const uint32_t s = __ldg(so + p);
#pragma unroll
            for (int v = 0; v < VPL; v++) add4(acc[v], ldg4(st + (size_t)s * D4 + lane + v * G));
        }
#pragma unroll
        for (int v = 0; v < VPL; v++) __stcs(out + bag * D4 + lane + v * G, acc[v]);
    }
}

// generic D (D/4 not a power-of-two multiple of 32): 32 lanes, strided columns
__global__ void __launch_bounds__(256) k_fwd_generic(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const int L = A.g.L, D4 = A.g.D / 4;
    const long long nbags = (long long)A.g.T * A.g.N;
    const int lane = threadIdx.x & 31;
    const float4 *st = reinterpret_cast<const float4 *>(A.storage);
    float4 *out = reinterpret_cast<float4 *>(A.pooled);
    for (long long bag = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; bag < nbags;
         bag += (long long)gridDim.x * (blockDim.x / 32)) {
        const uint32_t *so = A.bb.slot_of_occ + bag * L;
        for (int c = lane; c < D4; c += 32) {
            float4 acc = ldg4(st + (size_t)__ldg(so) * D4 + c);
            for (int p = 1; p < L; p++) add4(acc, ldg4(st + (size_t)__ldg(so + p) * D4 + c));
            out[bag * D4 + c] = acc;
        }
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

// Pass 1.  Work item = one chunk record of one table: up to CH occurrences of
// one unique row with their bag indices inline, so a chunk costs one record
// load, then its gradient rows (RB per round, all issued before folding),
// while the Storage row is prefetched.  Single-chunk rows (the common case)
// are updated here; hot rows write one fp64 partial per chunk, folded by
// k_bwd_hot (pass 2).
template <int G, int VPL>
__global__ void __launch_bounds__(256, 3) k_bwd(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ uint32_t s_pref[65];
    const int gpb = blockDim.x / G;
    const int lane = threadIdx.x % G;
    const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    constexpr int RB = VPL >= 4 ? 2 : (VPL == 2 ? 4 : 8);  // gradient rows per round
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.nchunks, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        for (uint32_t item = blockIdx.x * gpb + threadIdx.x / G; item < total; item += gridDim.x * gpb) {
            const int tl = find_table(s_pref, tcount, item);
            const int t = t0 + tl;
            const uint32_t c = item - s_pref[tl];
            const uint4 *rp = reinterpret_cast<const uint4 *>(A.bb.chunk_rec + (size_t)t * g.nc + c);
            uint4 q4[5];
            q4[0] = __ldg(rp);
            const uint32_t slot = q4[0].x, meta = q4[0].y;
            const uint32_t len = meta & 0xFFFFu;
            const bool multi = (meta >> 31) != 0;
#pragma unroll
            for (int k = 1; k < 5; k++) q4[k] = (uint32_t)(4 * k - 2) < len ? __ldg(rp + k) : make_uint4(0, 0, 0, 0);
            const uint32_t *bag = reinterpret_cast<const uint32_t *>(q4) + 2;
            const float4 *gb = grad + (size_t)t * g.N * D4 + lane;
            float4 w[VPL];
            float4 *wp = st + (size_t)slot * D4 + lane;
            if (!multi) {
#pragma unroll
                for (int v = 0; v < VPL; v++) w[v] = wp[v * G];
            }
            Acc4 acc[VPL];
#pragma unroll
            for (int v = 0; v < VPL; v++) acc[v] = Acc4{0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q0 = 0; q0 < CH; q0 += RB) {
                if ((uint32_t)q0 < len) {
                    float4 r[RB][VPL];
#pragma unroll
                    for (int q = 0; q < RB; q++)
                        if ((uint32_t)(q0 + q) < len)
#pragma unroll
                            for (int v = 0; v < VPL; v++) r[q][v] = ldg4(gb + (size_t)bag[q0 + q] * D4 + v * G);
#pragma unroll
                    for (int q = 0; q < RB; q++)
                        if ((uint32_t)(q0 + q) < len)
#pragma unroll
                            for (int v = 0; v < VPL; v++) acc_add(acc[v], r[q][v]);
                }
            }
            if (!multi) {
#pragma unroll
                for (int v = 0; v < VPL; v++) wp[v * G] = sgd(w[v], acc[v], A.lr);
            } else {
                double4 *part = reinterpret_cast<double4 *>(A.partial + ((size_t)t * g.nc + c) * g.D) + lane;
#pragma unroll
                for (int v = 0; v < VPL; v++) part[v * G] = make_double4(acc[v].x, acc[v].y, acc[v].z, acc[v].w);
            }
        }
    }
}

// generic D: one warp per chunk, strided columns
__global__ void __launch_bounds__(256) k_bwd_generic(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    const int lane = threadIdx.x & 31;
    const float4 *grad = reinterpret_cast<const float4 *>(A.grad);
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    const int wpb = blockDim.x / 32;
    for (int t = 0; t < g.T; t++) {
        const uint32_t total = A.bb.nchunks[t];
        for (uint32_t c = blockIdx.x * wpb + threadIdx.x / 32; c < total; c += gridDim.x * wpb) {
            const ChunkRec &rc = A.bb.chunk_rec[(size_t)t * g.nc + c];
            const uint32_t slot = rc.slot, len = rc.meta & 0xFFFFu;
            const bool multi = (rc.meta >> 31) != 0;
            double *part = A.partial + ((size_t)t * g.nc + c) * g.D;
            for (int col = lane; col < D4; col += 32) {
                Acc4 a{0.0, 0.0, 0.0, 0.0};
                for (uint32_t i = 0; i < len; i++)
                    acc_add(a, grad[((size_t)t * g.N + rc.bag[i]) * D4 + col]);
                if (!multi) st[(size_t)slot * D4 + col] = sgd(st[(size_t)slot * D4 + col], a, A.lr);
                else reinterpret_cast<double4 *>(part)[col] = make_double4(a.x, a.y, a.z, a.w);
            }
        }
    }
}

// Pass 2: one CTA per hot row folds its chunk partials: thread (p, col) sums
// partials p, p+PL, p+2PL, ... in order, then a fixed-shape tree over p
// (deterministic, independent of the grid), then the SGD update.
__global__ void __launch_bounds__(256) k_bwd_hot(TrainArgs A) {
    if (*A.err != NO_ERR) return;
    const Geometry g = A.g;
    const int D4 = g.D / 4;
    __shared__ double4 s_acc[256];
    __shared__ uint32_t s_pref[65];
    const int PL = D4 >= 256 ? 1 : 256 / D4;          // partial lanes per column (<= 256/D4)
    float4 *st = reinterpret_cast<float4 *>(A.storage);
    for (int t0 = 0; t0 < g.T; t0 += 64) {
        const int tcount = min(64, g.T - t0);
        table_prefix(A.bb.nhot, t0, tcount, s_pref);
        const uint32_t total = s_pref[tcount];
        for (uint32_t item = blockIdx.x; item < total; item += gridDim.x) {
            const int tl = find_table(s_pref, tcount, item);
            const int t = t0 + tl;
            const uint4 hr = A.bb.hot_rec[(size_t)t * g.nh + (item - s_pref[tl])];
            const uint32_t slot = hr.x, c0 = hr.y, nch = hr.z;
            const double4 *part = reinterpret_cast<const double4 *>(A.partial + ((size_t)t * g.nc + c0) * g.D);
            for (int col0 = 0; col0 < D4; col0 += 256 / PL) {
                const int p = threadIdx.x / (256 / PL > D4 ? D4 : 256 / PL);
                const int colw = 256 / PL > D4 ? D4 : 256 / PL;
                const int col = col0 + threadIdx.x % colw;
                Acc4 a{0.0, 0.0, 0.0, 0.0};
                if (p < PL && col < D4) {
                    uint32_t q = p;
                    for (; q + 3 * PL < nch; q += 4 * PL) {  // 4 partials in flight, folded in order
                        double4 d[4];
#pragma unroll
                        for (int k = 0; k < 4; k++) d[k] = part[(size_t)(q + k * PL) * D4 + col];
#pragma unroll
                        for (int k = 0; k < 4; k++) { a.x += d[k].x; a.y += d[k].y; a.z += d[k].z; a.w += d[k].w; }
                    }
                    for (; q < nch; q += PL) {
                        const double4 d = part[(size_t)q * D4 + col];
                        a.x += d.x; a.y += d.y; a.z += d.z; a.w += d.w;
                    }
                }
                __syncthreads();
                if (p < PL && col < D4) s_acc[p * colw + (col - col0)] = make_double4(a.x, a.y, a.z, a.w);
                __syncthreads();
                for (int half = 1; half < PL; half <<= 1) {   // fixed tree over p
                    if (p < PL && col < D4 && (p % (2 * half)) == 0 && p + half < PL) {
                        const double4 o = s_acc[(p + half) * colw + (col - col0)];
                        double4 &m = s_acc[p * colw + (col - col0)];
                        m.x += o.x; m.y += o.y; m.z += o.z; m.w += o.w;
                    }
                    __syncthreads();
                }
                if (p == 0 && col < D4) {
                    const double4 m = s_acc[col - col0];
                    float4 *wp = st + (size_t)slot * D4 + col;
                    *wp = sgd(*wp, Acc4{m.x, m.y, m.z, m.w}, A.lr);
                }
                __syncthreads();
            }
        }
    }
}

// -------------------------------------------------------------- surrogate
__global__ void __launch_bounds__(256) k_surrogate(const float4 *p, float4 *g, long long n4,
                                                   float gamma, float delta) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        float4 x = __ldcs(p + i), y;
        y.x = fmaf(gamma, x.x, delta);
        y.y = fmaf(gamma, x.y, delta);
        y.z = fmaf(gamma, x.z, delta);
        y.w = fmaf(gamma, x.w, delta);
        g[i] = y;
    }
}

// --------------------------------------------------------------- launchers
static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// resident CTAs of a kernel on the whole GPU (a persistent grid never waits
// for a second wave of a latency-bound kernel)
template <typename K>
static int resident_ctas(K kernel, int threads) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * num_sms();
}

template <int G, int VPL, typename K>
static void launch_sized(K kernel, long long groups, const TrainArgs &a, cudaStream_t s) {
    static std::unordered_map<const void *, int> caps;  // per kernel (not per signature)
    int &cap = caps[reinterpret_cast<const void *>(kernel)];
    if (!cap) cap = resident_ctas(kernel, 256);
    long long blocks = (groups + (256 / G) - 1) / (256 / G);
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    kernel<<<grid, 256, 0, s>>>(a);
}

#define SP_DISPATCH_D(D4, KERNEL, GROUPS, ARGS, STREAM)                                  \
    switch (D4) {                                                                         \
        case 1: launch_sized<1, 1>(KERNEL<1, 1>, GROUPS, ARGS, STREAM); break;            \
        case 2: launch_sized<2, 1>(KERNEL<2, 1>, GROUPS, ARGS, STREAM); break;            \
        case 4: launch_sized<4, 1>(KERNEL<4, 1>, GROUPS, ARGS, STREAM); break;            \
        case 8: launch_sized<8, 1>(KERNEL<8, 1>, GROUPS, ARGS, STREAM); break;            \
        case 16: launch_sized<16, 1>(KERNEL<16, 1>, GROUPS, ARGS, STREAM); break;         \
        case 32: launch_sized<32, 1>(KERNEL<32, 1>, GROUPS, ARGS, STREAM); break;         \
        case 64: launch_sized<32, 2>(KERNEL<32, 2>, GROUPS, ARGS, STREAM); break;         \
        case 128: launch_sized<32, 4>(KERNEL<32, 4>, GROUPS, ARGS, STREAM); break;        \
        case 256: launch_sized<32, 8>(KERNEL<32, 8>, GROUPS, ARGS, STREAM); break;        \
        default: launch_sized<32, 1>(KERNEL##_generic, GROUPS, ARGS, STREAM); break;      \
    }

cudaError_t launch_forward(const TrainArgs &a, cudaStream_t s) {
    const int D4 = a.g.D / 4;
    SP_DISPATCH_D(D4, k_fwd, (long long)a.g.T * a.g.N, a, s);
    return cudaGetLastError();
}

cudaError_t launch_backward(const TrainArgs &a, cudaStream_t s) {
    const int D4 = a.g.D / 4;
    // upper bound of work items: all chunks of all tables
    SP_DISPATCH_D(D4, k_bwd, (long long)a.g.T * a.g.nc, a, s);
    return cudaGetLastError();
}

cudaError_t launch_backward_hot(const TrainArgs &a, cudaStream_t s) {
    long long upper = (long long)a.g.T * a.g.nh;
    const long long cap = (long long)num_sms() * 4;
    int grid = (int)(upper < cap ? upper : cap);
    if (grid < 1) grid = 1;
    k_bwd_hot<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_surrogate(const float *pooled, float *grad, long long count, float gamma,
                             float delta, cudaStream_t s) {
    long long n4 = count / 4;
    long long blocks = (n4 + 255) / 256;
    const long long cap = (long long)num_sms() * 8;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    k_surrogate<<<grid, 256, 0, s>>>(reinterpret_cast<const float4 *>(pooled),
                                     reinterpret_cast<float4 *>(grad), n4, gamma, delta);
    return cudaGetLastError();
}

}  // namespace sp
