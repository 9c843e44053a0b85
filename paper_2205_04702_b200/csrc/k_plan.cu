// k_plan.cu — the [Plan] stage (Alg. 1) as ONE
// kernel launch per sp_plan call, one CTA per embedding table (one cache
// manager per table; tables are independent, so CTAs never
// synchronise with each other).
//
// CTA t of k_push does, for the batch B(j) entering the window and the batch
// B(b), b = j - F, leaving the look-ahead queue:
//   A1  ingest + range check of B(j)[t]
//   A2  dedup: sort (id, occurrence) pairs, mark heads, segment offsets
//       (Alg. 1 walks raw IDs; dedup first is equivalent, reading R5)
//   A3  backward work list: chunks of <= CH occurrences per unique
//   A4  future probe: slots of resident IDs of B(j) get next_need = j
//       (future window, RAW-4 rule; one-shot probe, reading R12)
//   B1  probe B(b): hit -> last_use = b (HoldMask |= MSB, Alg. 1)
//   B2  misses compacted in ascending ID order
//   B3  victims: walk the LRU log from its head; a slot is a candidate iff
//       last_use <= b-P-1 (past window) and next_need <= b
//       (future window); first |misses| candidates in (last_use, ID) order
//       (LRU, reading R8); too few -> SP_ERR_CAPACITY
//   B4  pair k-th miss with k-th victim (reading R6): Hit-Map / resident /
//       stamps updated, evict + fill lists for the transfer kernel
//   B5  append this batch's slots to the LRU log (compacting it if full)
//   B6  slot map for the Train stage (frozen at Plan, reading R13)
#include "sp_internal.cuh"

namespace sp {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exclusive block-wide scan of one u32 per thread; *total gets the sum.
// Contains __syncthreads: every thread of the CTA must call it.
__device__ uint32_t block_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t s_warp[PUSH_THREADS / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) s_warp[lane] = w;
    }
    __syncthreads();
    uint32_t pre = warp ? s_warp[warp - 1] : 0u;
    *total = s_warp[nw - 1];
    __syncthreads();
    return pre + x - v;
}

__device__ __forceinline__ void set_err(unsigned long long *err, long long b, int t, unsigned k) {
    atomicMin(err, err_key(b, t, k));
}

// ---- sort of (id << 32 | occ) keys, ascending ----------------------------
// small n: bitonic network in shared memory
__device__ void bitonic_sort_smem(uint64_t *key, int n_pad) {
    for (int k = 2; k <= n_pad; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < n_pad; i += blockDim.x) {
                int ixj = i ^ jj;
                if (ixj > i) {
                    uint64_t a = key[i], c = key[ixj];
                    bool up = (i & k) == 0;
                    if ((a > c) == up) { key[i] = c; key[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

// large n: stable LSD radix sort on the id (upper 32 bits), 8-bit digits,
// one CTA, ping-pong in global scratch.  Returns the buffer holding the result.
constexpr int RADIX_IPT = 8;
__device__ uint64_t *radix_sort_global(uint64_t *a, uint64_t *b, int n, int bits) {
    __shared__ uint32_t s_hist[256];
    __shared__ uint32_t s_wcnt[PUSH_THREADS / 32][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int tile = blockDim.x * RADIX_IPT;
    for (int sh = 32; sh < 32 + bits; sh += 8) {
        for (int d = threadIdx.x; d < 256; d += blockDim.x) s_hist[d] = 0;
        for (int w = 0; w < nw; w++)
            for (int d = threadIdx.x; d < 256; d += blockDim.x) s_wcnt[w][d] = 0;
        __syncthreads();
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
            int i = i0 + threadIdx.x;
            unsigned d = i < n ? (unsigned)((a[i] >> sh) & 255u) : 256u;
            unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && (peers & lanemask_lt()) == 0) atomicAdd(&s_hist[d], __popc(peers));
        }
        __syncthreads();
        // exclusive scan of the 256-bin histogram -> running bucket bases
        {
            uint32_t v = threadIdx.x < 256 ? s_hist[threadIdx.x] : 0u, tot;
            uint32_t ex = block_scan(v, &tot);
            if (threadIdx.x < 256) s_hist[threadIdx.x] = ex;
            __syncthreads();
        }
        for (int t0 = 0; t0 < n; t0 += tile) {
            uint64_t e[RADIX_IPT];
            uint32_t rk[RADIX_IPT];
            unsigned dg[RADIX_IPT];
            const int wbase = t0 + warp * 32 * RADIX_IPT;
#pragma unroll
            for (int r = 0; r < RADIX_IPT; r++) {
                int i = wbase + r * 32 + lane;
                e[r] = i < n ? a[i] : 0ull;
                dg[r] = i < n ? (unsigned)((e[r] >> sh) & 255u) : 256u;
                unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
                uint32_t base = dg[r] < 256u ? s_wcnt[warp][dg[r]] : 0u;
                rk[r] = base + __popc(peers & lanemask_lt());
                __syncwarp();
                if (dg[r] < 256u && (peers & lanemask_lt()) == 0) s_wcnt[warp][dg[r]] = base + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            for (int d = threadIdx.x; d < 256; d += blockDim.x) {
                uint32_t run = s_hist[d];
                for (int w = 0; w < nw; w++) {
                    uint32_t c = s_wcnt[w][d];
                    s_wcnt[w][d] = run;
                    run += c;
                }
                s_hist[d] = run;
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < RADIX_IPT; r++)
                if (dg[r] < 256u) b[s_wcnt[warp][dg[r]] + rk[r]] = e[r];
            __syncthreads();
            for (int w = 0; w < nw; w++)
                for (int d = threadIdx.x; d < 256; d += blockDim.x) s_wcnt[w][d] = 0;
            __syncthreads();
        }
        uint64_t *tmp = a; a = b; b = tmp;
    }
    return a;
}

__device__ int bit_width_u64(unsigned long long x) { return x ? 64 - __clzll(x) : 0; }

}  // namespace

__global__ void __launch_bounds__(PUSH_THREADS, 1) k_push(PushArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int t = blockIdx.x;
    const Geometry &g = A.g;
    const int n = g.n, tid = threadIdx.x;
    __shared__ uint32_t s_fail, s_got;
    __shared__ unsigned long long s_head, s_newhead, s_tail;
    if (*A.err != NO_ERR) return;  // poisoned: nothing more is planned
    const unsigned long long roff = A.row_off[t];
    const long long R = A.rows[t];

    // ------------------------------------------------------------ part A
    if (A.has_new) {
        BatchBufs &nb = A.nb;
        uint64_t *keys;
        const bool small = A.n_pad <= SMEM_SORT_MAX;
        uint64_t *gA = A.sort_tmp + (size_t)t * n;
        uint64_t *gB = A.sort_tmp + (size_t)g.T * n + (size_t)t * n;
        keys = small ? reinterpret_cast<uint64_t *>(smem_raw) : gA;
        // A1: ingest + range check; key = id << 32 | occurrence
        int bad = 0;
        for (int i = tid; i < (small ? A.n_pad : n); i += blockDim.x) {
            uint64_t k = ~0ull;
            if (i < n) {
                long long id = A.idx_i32 ? (long long)((const int32_t *)A.idx)[(size_t)t * n + i]
                                         : ((const long long *)A.idx)[(size_t)t * n + i];
                if (id < 0 || id >= R) { bad = 1; id = 0; }
                k = ((uint64_t)id << 32) | (uint32_t)i;
            }
            keys[i] = k;
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) set_err(A.err, A.j, t, DERR_INDEX);
            return;
        }
        // A2: sort + unique
        if (small) {
            bitonic_sort_smem(keys, A.n_pad);
        } else {
            int bits = bit_width_u64((unsigned long long)(R - 1));
            keys = radix_sort_global(gA, gB, n, bits);
            __syncthreads();
        }
        uint32_t *sorted_occ = nb.sorted_occ + (size_t)t * n;
        uint32_t *sorted_uid = nb.sorted_uid + (size_t)t * n;
        uint32_t *uniq_id = nb.uniq_id + (size_t)t * n;
        uint32_t *seg_off = nb.seg_off + (size_t)t * g.n1;
        uint32_t carry = 0;
        for (int i0 = 0; i0 < n; i0 += blockDim.x) {
            int i = i0 + tid;
            uint64_t k = i < n ? keys[i] : ~0ull;
            uint32_t id = (uint32_t)(k >> 32);
            uint32_t head = 0;
            if (i < n) head = (i == 0) || ((uint32_t)(keys[i - 1] >> 32) != id);
            uint32_t tot;
            uint32_t ex = block_scan(head, &tot);
            if (i < n) {
                uint32_t uid = carry + ex + head - 1;
                sorted_occ[i] = (uint32_t)k;
                sorted_uid[i] = uid;
                if (head) { uniq_id[uid] = id; seg_off[uid] = (uint32_t)i; }
            }
            carry += tot;
        }
        const uint32_t U = carry;
        if (tid == 0) { seg_off[U] = (uint32_t)n; nb.U[t] = U; }
        __syncthreads();
        // A3: backward chunks
        uint32_t *chunk_u = nb.chunk_u + (size_t)t * g.nc;
        uint32_t *chunk_first = nb.chunk_first + (size_t)t * n;
        carry = 0;
        for (uint32_t u0 = 0; u0 < U; u0 += blockDim.x) {
            uint32_t u = u0 + tid;
            uint32_t nch = 0;
            if (u < U) nch = (seg_off[u + 1] - seg_off[u] + CH - 1) / CH;
            uint32_t tot;
            uint32_t ex = block_scan(nch, &tot);
            if (u < U) {
                chunk_first[u] = carry + ex;
                for (uint32_t k = 0; k < nch; k++) chunk_u[carry + ex + k] = u;
            }
            carry += tot;
        }
        if (tid == 0) nb.nchunks[t] = carry;
        // A4: future probe of B(j)
        for (uint32_t u = tid; u < U; u += blockDim.x) {
            uint32_t s = A.hitmap[roff + uniq_id[u]];
            if (s != EMPTY) A.next_need[s] = (int32_t)A.j;
        }
        __syncthreads();
    }

    // ------------------------------------------------------------ part B
    if (!A.do_plan) return;
    BatchBufs &pb = A.pb;
    const long long b = A.b;
    const uint32_t Ub = pb.U[t];
    const uint32_t *uniq_id = pb.uniq_id + (size_t)t * n;
    uint32_t *slot_u = pb.slot_u + (size_t)t * n;
    uint8_t *hitf = pb.hit + (size_t)t * n;
    uint32_t *miss_u = A.miss_u + (size_t)t * n;
    uint32_t *victims = A.victims + (size_t)t * n;
    // B1 + B2: probe, hits stamped, misses compacted (ascending ID)
    uint32_t carry = 0, nhit = 0;
    for (uint32_t u0 = 0; u0 < Ub; u0 += blockDim.x) {
        uint32_t u = u0 + tid;
        uint32_t miss = 0;
        if (u < Ub) {
            uint32_t s = A.hitmap[roff + uniq_id[u]];
            if (s != EMPTY) {
                A.last_use[s] = (int32_t)b;
                slot_u[u] = s;
                hitf[u] = 1;
            } else {
                slot_u[u] = EMPTY;
                hitf[u] = 0;
                miss = 1;
            }
        }
        uint32_t tot;
        uint32_t ex = block_scan(miss, &tot);
        if (miss) miss_u[carry + ex] = u;
        carry += tot;
    }
    const uint32_t m = carry;
    nhit = Ub - m;
    __syncthreads();  // last_use of hits visible to the victim scan

    // B3: victim selection over the per-table LRU log
    const unsigned long long cap = A.log_cap[t], lbase = A.log_base[t];
    uint32_t *lslot = A.log_slot;
    int32_t *lstamp = A.log_stamp;
    if (tid == 0) {
        s_head = A.log_head[t];
        s_tail = A.log_tail[t];
        s_got = 0;
        s_fail = 0;
    }
    __syncthreads();
    const long long limit = b - A.P - 1;
    while (true) {
        const unsigned long long head = s_head, tail = s_tail;
        const uint32_t got = s_got;
        if (got >= m) break;
        unsigned long long pos = head + tid;
        bool inr = pos < tail;
        uint32_t slot = 0;
        int32_t stamp = 0;
        if (inr) {
            size_t ix = (size_t)(lbase + pos % cap);
            slot = lslot[ix];
            stamp = lstamp[ix];
        }
        bool elig = inr && (long long)stamp <= limit;
        bool cand = elig && A.last_use[slot] == stamp && (long long)A.next_need[slot] <= b;
        uint32_t n_elig, n_cand;
        (void)block_scan(elig ? 1u : 0u, &n_elig);
        uint32_t r = block_scan(cand ? 1u : 0u, &n_cand);
        const uint32_t need = m - got;
        if (cand && r < need) {
            victims[got + r] = slot;
            if (r == need - 1) s_newhead = pos + 1;
        }
        __syncthreads();
        if (tid == 0) {
            if (n_cand >= need) {
                s_got = m;
                s_head = s_newhead;
            } else {
                s_got = got + n_cand;
                s_head = head + n_elig;
                if (n_elig < blockDim.x) s_fail = 1;  // reached held entries or the tail
            }
        }
        __syncthreads();
        if (s_fail) break;
    }
    if (s_fail) {
        if (tid == 0) set_err(A.err, b, t, DERR_CAPACITY);
        return;
    }

    // B4: assignment (k-th miss <-> k-th victim)
    uint32_t *fill_slot = pb.fill_slot + (size_t)t * n;
    uint32_t *fill_row = pb.fill_row + (size_t)t * n;
    uint32_t *evict_row = pb.evict_row + (size_t)t * n;
    uint32_t nev = 0;
    for (uint32_t k = tid; k < m; k += blockDim.x) {
        uint32_t u = miss_u[k], s = victims[k], id = uniq_id[u];
        uint32_t old = A.resident[s];
        if (old != EMPTY) {
            A.hitmap[roff + old] = EMPTY;
            nev++;
        }
        A.hitmap[roff + id] = s;
        A.resident[s] = id;
        A.last_use[s] = (int32_t)b;
        A.next_need[s] = NEVER;
        slot_u[u] = s;
        fill_slot[k] = s;
        fill_row[k] = id;
        evict_row[k] = old;
    }
    uint32_t ev_total;
    (void)block_scan(nev, &ev_total);  // includes barriers: B4 writes visible below

    // B5: LRU log append (after an in-place compaction if it would overflow)
    unsigned long long head = s_head, tail = s_tail;
    if (tail - head + Ub > cap) {
        unsigned long long w = head;
        for (unsigned long long c0 = head; c0 < tail; c0 += blockDim.x) {
            unsigned long long pos = c0 + tid;
            bool inr = pos < tail;
            uint32_t slot = 0;
            int32_t stamp = 0;
            if (inr) {
                size_t ix = (size_t)(lbase + pos % cap);
                slot = lslot[ix];
                stamp = lstamp[ix];
            }
            bool keep = inr && A.last_use[slot] == stamp;
            uint32_t tot;
            uint32_t r = block_scan(keep ? 1u : 0u, &tot);  // all reads precede writes
            if (keep) {
                size_t ix = (size_t)(lbase + (w + r) % cap);
                lslot[ix] = slot;
                lstamp[ix] = stamp;
            }
            w += tot;
            __syncthreads();
        }
        tail = w;
    }
    for (uint32_t u = tid; u < Ub; u += blockDim.x) {
        size_t ix = (size_t)(lbase + (tail + u) % cap);
        lslot[ix] = slot_u[u];
        lstamp[ix] = (int32_t)b;
    }
    if (tid == 0) {
        A.log_head[t] = head;
        A.log_tail[t] = tail + Ub;
        pb.m[t] = m;
        uint32_t *st = pb.stats + 4 * t;
        st[0] = Ub; st[1] = nhit; st[2] = m; st[3] = ev_total;
        atomicAdd(&A.cum[0], (unsigned long long)Ub);
        atomicAdd(&A.cum[1], (unsigned long long)nhit);
        atomicAdd(&A.cum[2], (unsigned long long)m);
        atomicAdd(&A.cum[3], (unsigned long long)ev_total);
    }
    __syncthreads();  // slot_u complete (B4) before the slot map
    // B6: slot map for Train, frozen at Plan
    const uint32_t *sorted_occ = pb.sorted_occ + (size_t)t * n;
    const uint32_t *sorted_uid = pb.sorted_uid + (size_t)t * n;
    uint32_t *slot_of_occ = pb.slot_of_occ + (size_t)t * n;
    for (int i = tid; i < n; i += blockDim.x) slot_of_occ[sorted_occ[i]] = slot_u[sorted_uid[i]];
}

size_t push_smem_bytes(int n_pad) {
    return n_pad <= SMEM_SORT_MAX ? (size_t)n_pad * sizeof(uint64_t) : 0;
}

cudaError_t configure_push_kernel() {
    return cudaFuncSetAttribute(k_push, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(SMEM_SORT_MAX * sizeof(uint64_t)));
}

cudaError_t launch_push(const PushArgs &a, cudaStream_t s) {
    k_push<<<a.g.T, PUSH_THREADS, push_smem_bytes(a.n_pad), s>>>(a);
    return cudaGetLastError();
}

}  // namespace sp
