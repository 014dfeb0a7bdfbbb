/*
 * oracle/tsq_oracle.c -- TEST INFRASTRUCTURE ONLY (see tsq_oracle.h).
 *
 * Plain-C restatement of tsqsort's sort path:
 *   MitigationRng            pivot.py:25-54
 *   select_pivot ladder      pivot.py:66-248
 *   insertion_sort           smallsort.py:12-47
 *   stage driver _range      core.py:1643-1728
 *   stage partition contract core.py:944-967 (exits of _run_machine)
 *   sorted/reversed paths    core.py:991-1556 (result-preserving fast paths)
 * Instantiated for int32/uint32/int64/uint64/float32/float64 keys, with and
 * without a uint32 payload (records, key-only comparator).
 */
#include "tsq_oracle.h"

#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TSQO_TASK_MIN ((int64_t)1 << 15)

static inline int64_t tsqo_min3(int64_t x, int64_t y, int64_t z) {
  int64_t m = x < y ? x : y;
  return m < z ? m : z;
}

/* Python floor division (pivot.py uses //) */
static inline int64_t tsqo_floordiv(int64_t x, int64_t y) {
  int64_t q = x / y;
  if ((x % y != 0) && ((x < 0) != (y < 0))) q--;
  return q;
}

static void tsqo_stats_merge(tsqo_stats *dst, const tsqo_stats *src) {
  __atomic_fetch_add(&dst->comparisons, src->comparisons, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->array_writes, src->array_writes, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->scratch_writes, src->scratch_writes, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->stages, src->stages, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->handler_sorted, src->handler_sorted, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->handler_reversed, src->handler_reversed, __ATOMIC_RELAXED);
  __atomic_fetch_add(&dst->handler_fallbacks, src->handler_fallbacks, __ATOMIC_RELAXED);
  uint64_t cur = __atomic_load_n(&dst->max_depth, __ATOMIC_RELAXED);
  while (src->max_depth > cur &&
         !__atomic_compare_exchange_n(&dst->max_depth, &cur, src->max_depth, 1,
                                      __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
  }
}

#define KT int32_t
#define SFX _i32
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _i32p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

#define KT uint32_t
#define SFX _u32
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _u32p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

#define KT int64_t
#define SFX _i64
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _i64p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

#define KT uint64_t
#define SFX _u64
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _u64p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

#define KT float
#define SFX _f32
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _f32p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

#define KT double
#define SFX _f64
#define PAY 0
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#define SFX _f64p
#define PAY 1
#include "tsq_oracle_impl.inc"
#undef SFX
#undef PAY
#undef KT

void tsqo_default_config(tsqo_config *cfg) {
  cfg->insertion_threshold = 16;
  cfg->medof3_max_n = 70;
  cfg->medof5_max_n = 600;
  cfg->ninther_max_n = 60000;
  cfg->reverse_tolerance = 3;
  cfg->mitigation_enabled = 1;
  cfg->medof3_small_enabled = 1;
}

#define TSQO_RA 16807ull
#define TSQO_RM 2147483648ull

void tsqo_rng_init(tsqo_rng *rng, uint64_t seed) {
  rng->zgen = seed % TSQO_RM;
  rng->dran = 1.0;
  rng->dran2 = 2.0;
}

void tsqo_rng_next(tsqo_rng *rng) {
  rng->zgen = (TSQO_RA * rng->zgen) % TSQO_RM;
  rng->dran = 0.5 + (double)rng->zgen / (double)TSQO_RM;
  rng->dran2 = 1.0 + rng->dran;
}

int tsqo_sort(void *keys, uint32_t *payload, int64_t n, int key_dtype,
              const tsqo_config *cfg, tsqo_rng *rng, int threads,
              tsqo_stats *stats) {
  tsqo_stats local;
  if (!stats) stats = &local;
  memset(stats, 0, sizeof(*stats));
  if (key_dtype < TSQO_I32 || key_dtype > TSQO_F64) return -1;
  if (n <= 1) return 0;
  tsqo_rng_next(rng);   /* once per sort call, core.py:1602 */
  const double dran = rng->dran;
  if (threads < 1) threads = 1;
#define TSQO_DISPATCH(code, sfx, T)                                           \
  case code:                                                                  \
    if (payload)                                                              \
      sort_##sfx##p((T *)keys, payload, n, cfg, dran, threads, stats);        \
    else                                                                      \
      sort_##sfx((T *)keys, NULL, n, cfg, dran, threads, stats);              \
    break;
  switch (key_dtype) {
    TSQO_DISPATCH(TSQO_I32, _i32, int32_t)
    TSQO_DISPATCH(TSQO_U32, _u32, uint32_t)
    TSQO_DISPATCH(TSQO_I64, _i64, int64_t)
    TSQO_DISPATCH(TSQO_U64, _u64, uint64_t)
    TSQO_DISPATCH(TSQO_F32, _f32, float)
    TSQO_DISPATCH(TSQO_F64, _f64, double)
    default:
      return -1;
  }
#undef TSQO_DISPATCH
  return 0;
}

tsqo_decision tsqo_select_pivot_i64(int64_t *ar, int64_t a, int64_t b,
                                    const tsqo_config *cfg,
                                    const tsqo_rng *rng, uint64_t tally[3]) {
  tsqo_decision d;
  d.order_flag = select_pivot__i64(ar, NULL, a, b, cfg, rng->dran, tally);
  d.pi = (a + b) >> 1;
  d._pad = 0;
  return d;
}

void tsqo_insertion_sort_i64(int64_t *ar, int64_t lo, int64_t hi,
                             uint64_t tally[3]) {
  insertion__i64(ar, NULL, lo, hi, tally);
}

void tsqo_partition3_i64(int64_t *ar, int64_t a, int64_t b, int64_t p,
                         int64_t *new_l, int64_t *new_r) {
  uint64_t t[3] = {0, 0, 0};
  partition3__i64(ar, NULL, a, b, p, new_l, new_r, t);
}
