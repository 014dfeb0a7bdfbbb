/*
 * oracle/tsq_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's three-way partition sort (tsqsort 0.1.0,
 * /root/reference/pkg/src/tsqsort) used as the parity checker for the B200
 * path and as the CPU baseline arm of bench.py.  Only tests/, the smoke()
 * entry and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product (paper_1505_00558_b200) never links or calls it.
 *
 * Parity pin: tests/golden/ holds vectors produced by running the Python
 * reference itself (tests/golden/make_golden.py) -- pivot-ladder decisions
 * with their in-place side effects, RNG sequences, insertion-sort results and
 * whole-sort outputs -- and tests/test_oracle.py checks this restatement
 * against every one of them.
 */
#ifndef TSQ_ORACLE_H
#define TSQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes (same numbering as include/tsq.h, kept separate on purpose) */
enum {
  TSQO_NONE = 0, TSQO_I32 = 1, TSQO_U32 = 2, TSQO_I64 = 3, TSQO_U64 = 4,
  TSQO_F32 = 5, TSQO_F64 = 6
};

/* SortConfig, config.py:8-42 */
typedef struct {
  int64_t insertion_threshold;   /* 16 */
  int64_t medof3_max_n;          /* 70 */
  int64_t medof5_max_n;          /* 600 */
  int64_t ninther_max_n;         /* 60000 */
  int64_t reverse_tolerance;     /* 3 */
  int32_t mitigation_enabled;    /* 1 */
  int32_t medof3_small_enabled;  /* 1 */
} tsqo_config;

/* MitigationRng, pivot.py:25-49 */
typedef struct {
  uint64_t zgen;
  double dran;
  double dran2;
} tsqo_rng;

/* subset of SortStats, stats.py:33-70 (counts of this restatement, not of
 * the reference's two-hole machine) */
typedef struct {
  uint64_t comparisons;
  uint64_t array_writes;
  uint64_t scratch_writes;
  uint64_t max_depth;
  uint64_t stages;
  uint64_t handler_sorted;
  uint64_t handler_reversed;
  uint64_t handler_fallbacks;
} tsqo_stats;

/* PivotDecision, pivot.py:57-63 */
typedef struct {
  int64_t pi;
  int32_t order_flag;
  int32_t _pad;
} tsqo_decision;

void tsqo_default_config(tsqo_config *cfg);
void tsqo_rng_init(tsqo_rng *rng, uint64_t seed);   /* seed % 2^31 must be != 0 */
void tsqo_rng_next(tsqo_rng *rng);

/* Whole sort (Sorter.sort_with_stats, core.py:1586-1614), in place.
 * keys: n elements of key_dtype; payload: NULL or n uint32 (moved with keys,
 * compared by key only -- the key-only comparator of tests/test_core.py:93-103).
 * rng must be initialised; it is advanced once (core.py:1602).
 * threads > 1 runs independent sub-ranges as OpenMP tasks (results are the
 * same multiset order; counts are summed).  Returns 0, or -1 on bad dtype. */
int tsqo_sort(void *keys, uint32_t *payload, int64_t n, int key_dtype,
              const tsqo_config *cfg, tsqo_rng *rng, int threads,
              tsqo_stats *stats);

/* select_pivot (pivot.py:205-248) on int64 keys, in place; for pinning the
 * ladder and its sample side effects against the reference. */
tsqo_decision tsqo_select_pivot_i64(int64_t *ar, int64_t a, int64_t b,
                                    const tsqo_config *cfg,
                                    const tsqo_rng *rng, uint64_t tally[3]);

/* insertion_sort (smallsort.py:12-47) on int64 keys over [lo, hi]. */
void tsqo_insertion_sort_i64(int64_t *ar, int64_t lo, int64_t hi,
                             uint64_t tally[3]);

/* One stage's three-way partition of ar[a..b] around value p (the contract
 * of _run_machine's exits, core.py:944-967): returns new_l / new_r. */
void tsqo_partition3_i64(int64_t *ar, int64_t a, int64_t b, int64_t p,
                         int64_t *new_l, int64_t *new_r);

#ifdef __cplusplus
}
#endif
#endif
