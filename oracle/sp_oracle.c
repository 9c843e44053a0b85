/* sp_oracle.c — CPU ORACLE for ScratchPipe (arXiv 2205.04702).
 *
 * TEST INFRASTRUCTURE ONLY (see sp_oracle.h): never loaded by the product.
 * Plain, single-threaded, slow, obviously correct.  Compile with
 *   gcc -O2 -ffp-contract=off -fPIC -shared sp_oracle.c -lm
 * (no fast-math, no FMA contraction: every fmaf below is explicit).
 *
 * Precision: the paper's embeddings are fp32 ("x 4 Bytes"), so
 * tables, pooled vectors, surrogate gradients and the SGD update are fp32.
 * The coalesced gradient of a row is the fp32 rounding of the fp64 sum of its
 * duplicated gradients (reading R7): the paper fixes no summation
 * order, and an fp64 accumulator makes the result order-independent up to one
 * final rounding.
 */
#include "sp_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int32_t orc_version(void) { return 4; }

/* ------------------------------------------------------------------------ */
/* init generator: identical formula to workload/gen.py                      */
/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

float orc_init_value(uint64_t seed, int32_t t, int64_t row, int32_t col) {
    uint64_t h = splitmix64(seed);
    h = splitmix64(h ^ (uint64_t)(int64_t)t);
    h = splitmix64(h ^ (uint64_t)row);
    h = splitmix64(h ^ (uint64_t)(int64_t)col);
    double u24 = (double)(h >> 40);
    return (float)(u24 * (0.2 / 16777216.0) - 0.1);
}

/* ------------------------------------------------------------------------ */
/* Part A: uncached EmbeddingBag training + sparse SGD                       */
/*   forward  P:222-243 (gather by sparse ID, element-wise reduce = sum,     */
/*            reading R1), Fig. 2(a)                               */
/*   backward P:269-288 (gradient duplication + coalescing, then scatter     */
/*            update of the gathered rows), plain SGD (reading R2,           */
/*            P:1103-1106 "does not change the algorithmic properties")      */
/* Tables are materialised lazily from orc_init_value so that only touched   */
/* rows use memory.                                                          */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t rows;
    int32_t gid;          /* global table id the init values are keyed by */
    int64_t *pool_of_row; /* row -> index into pool (-1 = untouched) */
    float *pool;          /* [cap][D] */
    int64_t used, cap;
} lazy_table;

struct orc_train {
    int32_t T, D, N, L;
    int32_t allow_pad;   /* id == -1 means "no lookup" (only for the Fig. 2 pin) */
    int32_t bf16;        /* bf16 Storage (reading R28): values rounded at first touch and after each update */
    uint64_t seed;
    lazy_table *tab;
    /* scratch */
    float *pooled, *grad;
    int64_t *pairs; /* (id, occ) */
    double *acc;
    float *upd;
    int64_t *upd_row;
};

/* bf16 round-to-nearest-even of an fp32 value, returned widened to fp32
 * (reading R28; the bf16 format is fp32's top 16 bits: sign, 8-bit exponent,
 * 7-bit mantissa).  Ties go to the even mantissa; NaN stays NaN. */
float orc_bf16_round(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) {         /* inf or NaN: keep, quiet a NaN */
        if (u & 0x007fffffu) u |= 0x00400000u;
        u &= 0xffff0000u;
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);            /* round half to even on bit 16 */
        u &= 0xffff0000u;
    }
    memcpy(&x, &u, 4);
    return x;
}

void orc_bf16_round_array(int64_t n, const float *in, float *out) {
    for (int64_t i = 0; i < n; i++) out[i] = orc_bf16_round(in[i]);
}

static float *lazy_row(orc_train *o, int32_t t, int64_t row) {
    lazy_table *lt = &o->tab[t];
    int64_t k = lt->pool_of_row[row];
    if (k < 0) {
        if (lt->used == lt->cap) {
            int64_t nc = lt->cap ? lt->cap * 2 : 1024;
            lt->pool = (float *)realloc(lt->pool, (size_t)nc * o->D * sizeof(float));
            lt->cap = nc;
        }
        k = lt->used++;
        lt->pool_of_row[row] = k;
        for (int32_t j = 0; j < o->D; j++) {
            const float v = orc_init_value(o->seed, lt->gid, row, j);
            /* bf16 Storage: a row enters the scratchpad rounded (R28) */
            lt->pool[k * o->D + j] = o->bf16 ? orc_bf16_round(v) : v;
        }
    }
    return &lt->pool[k * o->D];
}

orc_train *orc_train_create(int32_t T, const int64_t *rows, int32_t D, int32_t N,
                            int32_t L, uint64_t init_seed) {
    if (T <= 0 || D <= 0 || N <= 0 || L <= 0) return NULL;
    orc_train *o = (orc_train *)calloc(1, sizeof(orc_train));
    o->T = T; o->D = D; o->N = N; o->L = L; o->seed = init_seed;
    o->tab = (lazy_table *)calloc((size_t)T, sizeof(lazy_table));
    for (int32_t t = 0; t < T; t++) {
        o->tab[t].rows = rows[t];
        o->tab[t].gid = t;
        o->tab[t].pool_of_row = (int64_t *)malloc((size_t)rows[t] * sizeof(int64_t));
        for (int64_t r = 0; r < rows[t]; r++) o->tab[t].pool_of_row[r] = -1;
    }
    int64_t n = (int64_t)N * L;
    o->pooled = (float *)malloc((size_t)N * D * sizeof(float));
    o->grad = (float *)malloc((size_t)N * D * sizeof(float));
    o->pairs = (int64_t *)malloc((size_t)n * 2 * sizeof(int64_t));
    o->acc = (double *)malloc((size_t)D * sizeof(double));
    o->upd = (float *)malloc((size_t)n * D * sizeof(float));
    o->upd_row = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    return o;
}

void orc_train_destroy(orc_train *o) {
    if (!o) return;
    for (int32_t t = 0; t < o->T; t++) {
        free(o->tab[t].pool_of_row);
        free(o->tab[t].pool);
    }
    free(o->tab); free(o->pooled); free(o->grad); free(o->pairs);
    free(o->acc); free(o->upd); free(o->upd_row); free(o);
}

static int cmp_pair(const void *a, const void *b) {
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;      /* sparse ID   */
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;      /* occurrence  */
    return 0;
}

int32_t orc_train_step(orc_train *o, const int64_t *ids, const float *grad_in,
                       float gamma, float delta, float eta, float *pooled_out,
                       int32_t *err_table) {
    const int32_t D = o->D, N = o->N, L = o->L;
    const int64_t n = (int64_t)N * L;
    /* range check first: a bad batch changes nothing */
    for (int32_t t = 0; t < o->T; t++)
        for (int64_t i = 0; i < n; i++) {
            int64_t id = ids[(int64_t)t * n + i];
            if (o->allow_pad && id == -1) continue;
            if (id < 0 || id >= o->tab[t].rows) {
                if (err_table) *err_table = t;
                return ORC_ERR_INDEX;
            }
        }
    for (int32_t t = 0; t < o->T; t++) {   /* tables are independent */
        const int64_t *tid = ids + (int64_t)t * n;
        /* forward: pooled[s] = E[id(s,0)] + E[id(s,1)] + ... (left fold, p ascending) */
        for (int32_t s = 0; s < N; s++) {
            float *ps = &o->pooled[(int64_t)s * D];
            int32_t first = 1;
            for (int32_t j = 0; j < D; j++) ps[j] = 0.0f;     /* empty bag -> zero vector */
            for (int32_t p = 0; p < L; p++) {
                int64_t id = tid[(int64_t)s * L + p];
                if (id == -1) continue;                        /* padding (allow_pad only) */
                const float *e = lazy_row(o, t, id);
                for (int32_t j = 0; j < D; j++) ps[j] = first ? e[j] : ps[j] + e[j];
                first = 0;
            }
        }
        if (pooled_out) memcpy(pooled_out + (int64_t)t * N * D, o->pooled, (size_t)N * D * sizeof(float));
        /* gradients G[s] routed back from the MLP, one per reduced embedding */
        for (int64_t k = 0; k < (int64_t)N * D; k++)
            o->grad[k] = grad_in ? grad_in[(int64_t)t * N * D + k]
                                 : fmaf(gamma, o->pooled[k], delta);
        /* duplication + coalescing: per unique row, sum the gradients of
         * every occurrence, occurrences in ascending (s,p) order, fp64 accumulator */
        int64_t np_ = 0;
        for (int64_t i = 0; i < n; i++) {
            if (tid[i] == -1) continue;                        /* padding (allow_pad only) */
            o->pairs[2 * np_] = tid[i]; o->pairs[2 * np_ + 1] = i; np_++;
        }
        qsort(o->pairs, (size_t)np_, 2 * sizeof(int64_t), cmp_pair);
        int64_t nu = 0;
        for (int64_t i = 0; i < np_;) {
            int64_t row = o->pairs[2 * i];
            for (int32_t j = 0; j < D; j++) o->acc[j] = 0.0;
            int64_t k = i;
            for (; k < np_ && o->pairs[2 * k] == row; k++) {
                int64_t s = o->pairs[2 * k + 1] / L;
                for (int32_t j = 0; j < D; j++) o->acc[j] += (double)o->grad[s * D + j];
            }
            for (int32_t j = 0; j < D; j++) o->upd[nu * D + j] = (float)o->acc[j];
            o->upd_row[nu++] = row;
            i = k;
        }
        /* scatter update after all reads of this batch (RAW-1 honoured) */
        for (int64_t u = 0; u < nu; u++) {
            float *e = lazy_row(o, t, o->upd_row[u]);
            for (int32_t j = 0; j < D; j++) {
                const float w = fmaf(-eta, o->upd[u * D + j], e[j]);
                e[j] = o->bf16 ? orc_bf16_round(w) : w;   /* bf16 Storage: the update is stored rounded (R28) */
            }
        }
    }
    return ORC_OK;
}

void orc_train_set_padding(orc_train *o, int32_t allow) { o->allow_pad = allow; }
void orc_train_set_bf16(orc_train *o, int32_t on) { o->bf16 = on; }

/* Table-wise sharding (one cache-manager instance per table):
 * a trainer holding a subset of the tables keys their initial values by the
 * GLOBAL table id, so per-rank trainers together equal one trainer over all
 * tables. */
void orc_train_set_table_ids(orc_train *o, const int32_t *gid) {
    for (int32_t t = 0; t < o->T; t++) o->tab[t].gid = gid[t];
}

void orc_train_get_row(const orc_train *o, int32_t t, int64_t row, float *out) {
    const lazy_table *lt = &o->tab[t];
    int64_t k = lt->pool_of_row[row];
    for (int32_t j = 0; j < o->D; j++)
        out[j] = k < 0 ? orc_init_value(o->seed, lt->gid, row, j) : lt->pool[k * o->D + j];
}

int64_t orc_train_touched(const orc_train *o, int32_t t, int64_t *out, int64_t cap) {
    int64_t c = 0;
    for (int64_t r = 0; r < o->tab[t].rows; r++)
        if (o->tab[t].pool_of_row[r] >= 0) {
            if (c < cap) out[c] = r;
            c++;
        }
    return c;
}

/* ------------------------------------------------------------------------ */
/* Part B: reference scratchpad policy (IDs only), one manager per table     */
/* (P:1354-1356).  State per slot: resident ID (-1 vacant) and last_use =    */
/* the last Plan index that hit or filled the slot (reading R8; vacant =     */
/* -infinity, reading R9).  Hit-Map = dense row -> slot array.   */
/* For each b (Alg. 1, window rules P:840-896):                    */
/*   1. U_b = sorted unique IDs of B(b)[t]        (dedup first, reading R5)  */
/*   2. split into hits and misses (ascending)    (Alg. 1)          */
/*   3. hits: last_use = b                        (HoldMask |= MSB)          */
/*   4. future set = slots of resident IDs of B(b+1..min(b+F,nb-1))          */
/*                                                (RAW-4 rule)    */
/*   5. candidates = slots with last_use <= b-P-1 (past rule)     */
/*      and not in the future set; order by (last_use, resident ID, slot)   */
/*      (LRU; tie rule R8); fewer than |misses| -> CAPACITY          */
/*      (reading R11)                                           */
/*   6. pair k-th smallest miss with k-th candidate (reading R6); the old    */
/*      resident of a non-vacant victim is evicted; Hit-Map/resident updated;*/
/*      last_use = b                                                         */
/* ------------------------------------------------------------------------ */
#define ORC_VACANT INT64_MIN

/* Replacement-policy variants ("changing the GPU scratchpad's
 * replacement policy from our default LRU ... to a random eviction or LFU";
 * readings R23-R25 in DESIGN.md).  In every variant the CANDIDATES are the
 * same (past window, future window, not pinned); only their order differs:
 *   LRU     ascending (last_use, resident ID, slot)                  (R8)
 *   LFU     ascending (freq, last_use, resident ID, slot); freq = 1 at fill,
 *           +1 per Plan that hits the slot, saturating at ORC_LFU_FMAX (R24)
 *   RANDOM  vacant candidates first (ascending slot, R9), then the draw
 *           sequence s_i = H(seed, t, b, i) mod O, i = 0, 1, ..., where O is
 *           the number of occupied dynamic slots at the start of Plan(b)
 *           (occupied slots are [0, O): vacant ones are filled lowest
 *           first), keeping each occupied candidate the first time it is
 *           drawn: a uniformly random ordering of the occupied candidates
 *           (R23).  H = splitmix64 chain sm(sm(sm(sm(seed ^ RAND) ^ t) ^ b) ^ i).
 * Pinned slots (static top-N partition, reading R26): the
 * last `count` slots of a table hold rows loaded before the first Plan and
 * are never candidates. */
typedef struct {
    int64_t rows, S;
    int64_t S_dyn;         /* slots [0, S_dyn) are dynamic, [S_dyn, S) pinned */
    int64_t *slot_of_row;  /* Hit-Map: row -> slot or -1 */
    int64_t *resident;     /* slot -> row or -1 */
    int64_t *last_use;     /* slot -> stamp (ORC_VACANT if never used) */
    int64_t *freq;         /* slot -> LFU use count (0 vacant) */
    uint8_t *future;       /* scratch: slot in future set */
    uint8_t *taken;        /* scratch: slot drawn this Plan (RANDOM) */
    int64_t *cand;         /* scratch: candidate (key, last_use, resident, slot) tuples */
} pol_table;

struct orc_policy {
    int32_t T, P, F;
    int32_t full_sort;     /* 1: always sort every candidate (cross-check mode) */
    int32_t kind;          /* ORC_POL_* */
    uint64_t seed;         /* RANDOM draw seed */
    int32_t allow_pad;     /* id == -1 is "no lookup" (ragged bags, R27) */
    int32_t planned;       /* a Plan has run (pinning no longer allowed) */
    pol_table *tab;
    int64_t *ids;          /* scratch for sorting a batch */
};

orc_policy *orc_policy_create(int32_t T, const int64_t *rows, const int64_t *slots,
                              int32_t P, int32_t F) {
    if (T <= 0 || P < 0 || F < 0) return NULL;
    orc_policy *p = (orc_policy *)calloc(1, sizeof(orc_policy));
    p->T = T; p->P = P; p->F = F;
    p->tab = (pol_table *)calloc((size_t)T, sizeof(pol_table));
    for (int32_t t = 0; t < T; t++) {
        pol_table *pt = &p->tab[t];
        pt->rows = rows[t]; pt->S = slots[t];
        pt->slot_of_row = (int64_t *)malloc((size_t)rows[t] * sizeof(int64_t));
        for (int64_t r = 0; r < rows[t]; r++) pt->slot_of_row[r] = -1;
        pt->S_dyn = slots[t];
        pt->resident = (int64_t *)malloc((size_t)slots[t] * sizeof(int64_t));
        pt->last_use = (int64_t *)malloc((size_t)slots[t] * sizeof(int64_t));
        pt->freq = (int64_t *)calloc((size_t)slots[t], sizeof(int64_t));
        pt->future = (uint8_t *)calloc((size_t)slots[t], 1);
        pt->taken = (uint8_t *)calloc((size_t)slots[t], 1);
        pt->cand = (int64_t *)malloc((size_t)slots[t] * 4 * sizeof(int64_t));
        for (int64_t s = 0; s < slots[t]; s++) { pt->resident[s] = -1; pt->last_use[s] = ORC_VACANT; }
    }
    return p;
}

void orc_policy_destroy(orc_policy *p) {
    if (!p) return;
    for (int32_t t = 0; t < p->T; t++) {
        pol_table *pt = &p->tab[t];
        free(pt->slot_of_row); free(pt->resident); free(pt->last_use); free(pt->freq);
        free(pt->future); free(pt->taken); free(pt->cand);
    }
    free(p->tab); free(p->ids); free(p);
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

#define CW 4  /* candidate tuple: (policy key, last_use, resident ID, slot) */
static int cmp_cand(const void *a, const void *b) {
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    for (int i = 0; i < CW; i++)
        if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

/* move the k smallest tuples of c[0..n) to c[0..k), ascending (bounded max-heap) */
static void heap_sift(int64_t *h, int64_t k, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < k && cmp_cand(&h[CW * l], &h[CW * m]) > 0) m = l;
        if (r < k && cmp_cand(&h[CW * r], &h[CW * m]) > 0) m = r;
        if (m == i) return;
        for (int j = 0; j < CW; j++) { int64_t x = h[CW * i + j]; h[CW * i + j] = h[CW * m + j]; h[CW * m + j] = x; }
        i = m;
    }
}

static void select_smallest(int64_t *c, int64_t n, int64_t k) {
    for (int64_t i = k / 2 - 1; i >= 0; i--) heap_sift(c, k, i);
    for (int64_t i = k; i < n; i++)
        if (cmp_cand(&c[CW * i], &c[0]) < 0) {
            for (int j = 0; j < CW; j++) c[j] = c[CW * i + j];
            heap_sift(c, k, 0);
        }
    qsort(c, (size_t)k, CW * sizeof(int64_t), cmp_cand);
}

/* RANDOM draw H(seed, t, b, i) (reading R23; its own copy of splitmix64) */
static uint64_t rand_draw(uint64_t seed, int32_t t, int64_t b, int64_t i) {
    uint64_t h = splitmix64(seed ^ 0x52414E44ull);  /* "RAND" */
    h = splitmix64(h ^ (uint64_t)(int64_t)t);
    h = splitmix64(h ^ (uint64_t)b);
    return splitmix64(h ^ (uint64_t)i);
}

void orc_policy_set_kind(orc_policy *p, int32_t kind, uint64_t seed) { p->kind = kind; p->seed = seed; }
void orc_policy_set_padding(orc_policy *p, int32_t allow) { p->allow_pad = allow; }

/* Static partition (R26): rows ids[0..count) (distinct, in range) occupy the
 * table's last `count` slots, in the given order, before the first Plan. */
int32_t orc_policy_pin(orc_policy *p, int32_t t, const int64_t *ids, int64_t count) {
    pol_table *pt = &p->tab[t];
    if (p->planned || count < 0 || count > pt->S || pt->S_dyn != pt->S) return ORC_ERR_ARG;
    int64_t base = pt->S - count;
    for (int64_t k = 0; k < count; k++) {
        int64_t id = ids[k];
        if (id < 0 || id >= pt->rows || pt->slot_of_row[id] >= 0) return ORC_ERR_ARG;
        pt->slot_of_row[id] = base + k;
        pt->resident[base + k] = id;
    }
    pt->S_dyn = base;
    return ORC_OK;
}

void orc_policy_set_full_sort(orc_policy *p, int32_t on) { p->full_sort = on; }

int32_t orc_policy_plan(orc_policy *p, const int64_t *trace, int64_t nb, int32_t N,
                        int32_t L, int64_t b, int64_t *counts, int64_t *uniq,
                        int64_t *slot, int64_t *hit, int64_t *evicted,
                        int32_t *err_table) {
    const int64_t n = (int64_t)N * L;
    const int64_t T = p->T;
    if (b < 0 || b >= nb) return ORC_ERR_ARG;
    if (!p->ids) p->ids = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    p->planned = 1;
    for (int32_t t = 0; t < T; t++) {
        pol_table *pt = &p->tab[t];
        const int64_t *bt = trace + ((int64_t)b * T + t) * n;
        /* 1. U_b (with padding, -1 entries are not lookups) */
        int64_t nr = 0;
        for (int64_t i = 0; i < n; i++) {
            if (p->allow_pad && bt[i] == -1) continue;
            if (bt[i] < 0 || bt[i] >= pt->rows) { if (err_table) *err_table = t; return ORC_ERR_INDEX; }
            p->ids[nr++] = bt[i];
        }
        qsort(p->ids, (size_t)nr, sizeof(int64_t), cmp_i64);
        int64_t U = 0;
        for (int64_t i = 0; i < nr; i++)
            if (i == 0 || p->ids[i] != p->ids[i - 1]) p->ids[U++] = p->ids[i];
        int64_t *ou = uniq + (int64_t)t * n, *os = slot + (int64_t)t * n;
        int64_t *oh = hit + (int64_t)t * n, *oe = evicted + (int64_t)t * n;
        /* 2./3. hits and misses */
        int64_t nh = 0, nm = 0;
        for (int64_t k = 0; k < U; k++) {
            int64_t id = p->ids[k];
            ou[k] = id; oe[k] = -1;
            int64_t s = pt->slot_of_row[id];
            if (s >= 0) {
                oh[k] = 1; os[k] = s; pt->last_use[s] = b; nh++;
                if (pt->freq[s] < ORC_LFU_FMAX) pt->freq[s]++;
            }
            else { oh[k] = 0; os[k] = -1; nm++; }
        }
        /* 4. future set */
        memset(pt->future, 0, (size_t)pt->S);
        for (int64_t f = 1; f <= p->F && b + f < nb; f++) {
            const int64_t *ft = trace + ((int64_t)(b + f) * T + t) * n;
            for (int64_t i = 0; i < n; i++) {
                if (ft[i] < 0 || ft[i] >= pt->rows) continue; /* padding, or reported when planned */
                int64_t s = pt->slot_of_row[ft[i]];
                if (s >= 0) pt->future[s] = 1;
            }
        }
        /* 5. candidates (past window, future window, dynamic slots only), each
         * with its policy key: LRU 0, LFU freq, RANDOM 0 for vacant / 1 occupied */
        int64_t nc = 0, nvac = 0, occ = 0;
        for (int64_t s = 0; s < pt->S_dyn; s++) {
            int64_t lu = pt->last_use[s];
            if (pt->resident[s] >= 0) occ++;
            if (lu != ORC_VACANT && lu > b - p->P - 1) continue;
            if (pt->future[s]) continue;
            int64_t key = 0;
            if (p->kind == ORC_POL_LFU) key = pt->freq[s];
            else if (p->kind == ORC_POL_RANDOM) key = pt->resident[s] >= 0 ? 1 : 0;
            int64_t *c = &pt->cand[CW * nc];
            c[0] = key; c[1] = lu; c[2] = pt->resident[s]; c[3] = s;
            nc++;
            if (pt->resident[s] < 0) nvac++;
        }
        if (nc < nm) { if (err_table) *err_table = t; return ORC_ERR_CAPACITY; }
        int64_t *vic = pt->cand;  /* victims in order: slot of the k-th = vic[CW*k + 3] */
        if (p->kind == ORC_POL_RANDOM) {
            /* occupied slots are [0, occ): vacant slots are filled lowest first */
            for (int64_t s = 0; s < pt->S_dyn; s++)
                if ((s < occ) != (pt->resident[s] >= 0)) return ORC_ERR_ARG;
            /* vacant candidates first (ascending slot), then draw order */
            qsort(pt->cand, (size_t)nc, CW * sizeof(int64_t), cmp_cand);  /* vacant ones lead */
            int64_t got = nvac < nm ? nvac : nm;
            for (int64_t i = 0; got < nm; i++) {
                int64_t s = (int64_t)(rand_draw(p->seed, t, b, i) % (uint64_t)occ);
                int64_t lu = pt->last_use[s];
                if (lu != ORC_VACANT && lu > b - p->P - 1) continue;
                if (pt->future[s] || pt->taken[s]) continue;
                pt->taken[s] = 1;
                vic[CW * got + 3] = s;  /* (only the slot column is read below) */
                got++;
            }
            for (int64_t k = nvac < nm ? nvac : nm; k < nm; k++) pt->taken[vic[CW * k + 3]] = 0;
        } else {
            /* the first nm candidates in (key, last_use, resident, slot) order: the
             * order is total, so selecting the nm smallest and sorting them equals
             * sorting all */
            if (!p->full_sort && nm > 0 && nm * 16 < nc) select_smallest(pt->cand, nc, nm);
            else qsort(pt->cand, (size_t)nc, CW * sizeof(int64_t), cmp_cand);
        }
        /* 6. pair k-th miss with k-th victim */
        int64_t ne = 0, v = 0;
        for (int64_t k = 0; k < U; k++) {
            if (oh[k]) continue;
            int64_t s = vic[CW * v + 3];
            v++;
            int64_t old = pt->resident[s];
            if (old >= 0) { pt->slot_of_row[old] = -1; oe[k] = old; ne++; }
            pt->slot_of_row[ou[k]] = s;
            pt->resident[s] = ou[k];
            pt->last_use[s] = b;
            pt->freq[s] = 1;
            os[k] = s;
        }
        counts[4 * t + 0] = U; counts[4 * t + 1] = nh;
        counts[4 * t + 2] = nm; counts[4 * t + 3] = ne;
    }
    return ORC_OK;
}

int64_t orc_policy_resident(const orc_policy *p, int32_t t, int64_t *out, int64_t cap) {
    const pol_table *pt = &p->tab[t];
    int64_t c = 0;
    for (int64_t r = 0; r < pt->rows; r++)  /* ascending row order = sorted */
        if (pt->slot_of_row[r] >= 0) { if (c < cap) out[c] = r; c++; }
    return c;
}

void orc_policy_slots(const orc_policy *p, int32_t t, int64_t *resident, int64_t *last_use) {
    const pol_table *pt = &p->tab[t];
    for (int64_t s = 0; s < pt->S; s++) {
        resident[s] = pt->resident[s];
        last_use[s] = pt->last_use[s];
    }
}

void orc_policy_freq(const orc_policy *p, int32_t t, int64_t *freq) {
    const pol_table *pt = &p->tab[t];
    for (int64_t s = 0; s < pt->S; s++) freq[s] = pt->freq[s];
}

/* element-wise fp32 fmaf (C99 fmaf: one rounding) for the Python-side Part C */
void orc_fmaf_array(int64_t n, const float *a, const float *b, const float *c, float *out) {
    for (int64_t i = 0; i < n; i++) out[i] = fmaf(a[i], b[i], c[i]);
}
