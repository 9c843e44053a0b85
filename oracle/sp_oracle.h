/* sp_oracle.h — CPU ORACLE for ScratchPipe (arXiv 2205.04702).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product (paper_2205_04702_b200/, include/scratchpipe.h) shares no code,
 * header, table or constant with this file and never loads it.
 *
 * Citations: P:<n> = /root/reference/PAPER.md line n (LaTeX source of the
 * paper); S:<n> = SPEC.md line n; SURVEY §8(c) readings are listed in DESIGN.md.
 *
 * Parts:
 *   A  uncached EmbeddingBag training with sparse SGD (ground truth)
 *   B  reference scratchpad policy (IDs only): Hit-Map, past/future window,
 *      LRU victim choice, capacity error
 *   (Part C, the cycle-level pipeline with values and hazard checker, is
 *    oracle/pipeline.py: small cases only.)
 */
#ifndef SP_ORACLE_H
#define SP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_CAPACITY 2
#define ORC_ERR_INDEX 3

int32_t orc_version(void);

/* init(seed,t,row,col): same counter-based generator as workload/gen.py. */
float orc_init_value(uint64_t seed, int32_t t, int64_t row, int32_t col);

/* ---------------- Part A ---------------- */
typedef struct orc_train orc_train;
orc_train *orc_train_create(int32_t T, const int64_t *rows, int32_t D, int32_t N,
                            int32_t L, uint64_t init_seed);
void orc_train_destroy(orc_train *o);
/* One training iteration over every table.  ids: [T][N][L] int64.
 * grad_in: [T][N][D] pooled gradients, or NULL -> surrogate
 * g = fmaf(gamma, pooled, delta).  pooled_out: [T][N][D] or NULL.
 * Returns ORC_OK or ORC_ERR_INDEX (*err_table set). */
int32_t orc_train_step(orc_train *o, const int64_t *ids, const float *grad_in,
                       float gamma, float delta, float eta, float *pooled_out,
                       int32_t *err_table);
void orc_train_get_row(const orc_train *o, int32_t t, int64_t row, float *out);
/* allow id == -1 as "no lookup" (ragged bags; used only to pin Fig. 2) */
void orc_train_set_padding(orc_train *o, int32_t allow);
/* bf16 Storage (reading R28): every value rounded to bf16 (round to nearest
 * even) when its row is first touched and after every update; the forward and
 * the coalescing stay fp32 / fp64.  Set before the first step. */
void orc_train_set_bf16(orc_train *o, int32_t on);
float orc_bf16_round(float x);
void orc_bf16_round_array(int64_t n, const float *in, float *out);
/* init values of local table t keyed by global table id gid[t] (sharding) */
void orc_train_set_table_ids(orc_train *o, const int32_t *gid);
/* sorted list of rows ever touched in table t; returns count (writes <= cap) */
int64_t orc_train_touched(const orc_train *o, int32_t t, int64_t *out, int64_t cap);

/* ---------------- Part B ---------------- */
typedef struct orc_policy orc_policy;
orc_policy *orc_policy_create(int32_t T, const int64_t *rows, const int64_t *slots,
                              int32_t P, int32_t F);
void orc_policy_destroy(orc_policy *p);
/* Plan batch b of the trace [nb][T][N][L].  Per table t, with n = N*L:
 *   counts[t*4+0..3] = U, hits, misses, evictions
 *   uniq[t*n + k]    = k-th smallest unique ID of B(b)[t]       (k < U)
 *   slot[t*n + k]    = its Storage slot after this Plan
 *   hit[t*n + k]     = 1 if it hit the Hit-Map, 0 if it missed
 *   evicted[t*n + k] = for a miss: the ID previously resident in its
 *                      victim slot, or -1 if the slot was vacant; -1 for hits
 * Returns ORC_OK, ORC_ERR_CAPACITY (*err_table set) or ORC_ERR_INDEX. */
int32_t orc_policy_plan(orc_policy *p, const int64_t *trace, int64_t nb, int32_t N,
                        int32_t L, int64_t b, int64_t *counts, int64_t *uniq,
                        int64_t *slot, int64_t *hit, int64_t *evicted,
                        int32_t *err_table);
/* 1 = sort every candidate each Plan (cross-check of the default partial
 * selection of the |misses| smallest, which yields the same victims) */
void orc_policy_set_full_sort(orc_policy *p, int32_t on);
/* Replacement-policy variants (R23-R25): the
 * candidates are the same in every variant, only their order differs. */
#define ORC_POL_LRU 0
#define ORC_POL_RANDOM 1
#define ORC_POL_LFU 2
#define ORC_LFU_FMAX 8   /* LFU use counts saturate here (R24) */
void orc_policy_set_kind(orc_policy *p, int32_t kind, uint64_t seed);
/* id == -1 is "no lookup" (ragged bags as -1 padding, R27) */
void orc_policy_set_padding(orc_policy *p, int32_t allow);
/* static partition (R26): ids occupy the last `count` slots of table t,
 * never evicted; only before the first Plan */
int32_t orc_policy_pin(orc_policy *p, int32_t t, const int64_t *ids, int64_t count);
/* LFU use count per slot of table t */
void orc_policy_freq(const orc_policy *p, int32_t t, int64_t *freq);
/* sorted resident IDs of table t; returns count */
int64_t orc_policy_resident(const orc_policy *p, int32_t t, int64_t *out, int64_t cap);
/* slot-level view: resident id (-1 vacant) and last_use stamp per slot */
void orc_policy_slots(const orc_policy *p, int32_t t, int64_t *resident, int64_t *last_use);

/* element-wise C99 fmaf, used by the Python Part C (oracle/pipeline.py) */
void orc_fmaf_array(int64_t n, const float *a, const float *b, const float *c, float *out);

#ifdef __cplusplus
}
#endif
#endif
