/*
 * include/tsq.h -- C ABI of the B200 three-way partition sort
 * (libtsq_b200.so, built from paper_1505_00558_b200/csrc/).
 *
 * Drop-in boundary.  The reference (tsqsort 0.1.0, pure Python) has no FFI;
 * its sort path is the Python API below, and each entry point here is what a
 * native binding of that API calls (the ctypes stub a maintainer would add to
 * the reference is shown in INTEGRATION.md):
 *
 *   tsq_sort              <- Sorter.sort_with_stats / tsqsort.sort
 *                            (/root/reference/pkg/src/tsqsort/core.py:1586-1614,
 *                             core.py:1757-1770); in place, returns counters
 *   tsq_workspace_*       <- TempStore.ensure / release and
 *                            Sorter.free_temp_storage (core.py:81-104,
 *                            core.py:1616-1620): a retained, high-water
 *                            device workspace owned by one sorter
 *   tsq_partition_segment <- the per-stage contract entry points
 *                            init_stage .. copy_back (core.py:1789-1870):
 *                            one three-way partition of one segment around a
 *                            given pivot, returning the stage bounds
 *   tsq_select_pivot      <- select_pivot (pivot.py:205-248): the device
 *                            pivot-sampling kernel on one segment
 *   tsq_apply_permutation <- bigelem._apply / apply_permutation
 *                            (bigelem.py:48-86): the late-swap move of
 *                            large elements, one gather pass
 *
 * Conventions: plain pointers and sizes; `keys`/`payload` are DEVICE
 * pointers owned by the caller and sorted in place; work is enqueued on the
 * given cudaStream_t (passed as void*, NULL = legacy default stream); calls
 * that return statistics synchronise that stream.  One call in flight per
 * workspace (the reference's non-reentrancy rule, core.py:1589-1590).
 * Keys compare with the native order of their type (IEEE order for floats,
 * -0.0 placed before +0.0, NaNs after +inf / before -inf by sign bit).
 */
#ifndef TSQ_H
#define TSQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSQ_ABI_VERSION 2

typedef enum {
  TSQ_OK = 0,
  TSQ_ERR_ALLOC = 1,              /* -> TempAllocationError (core.py:46-47) */
  TSQ_ERR_UNSUPPORTED_DTYPE = 2,  /* -> TypeError */
  TSQ_ERR_CUDA = 3,               /* -> RuntimeError */
  TSQ_ERR_DEPTH_EXCEEDED = 4,     /* level limit reached (cannot happen: beyond the depth
                                   * guard segments split at their key-bound midpoint) */
  TSQ_ERR_INVALID = 5,            /* -> ValueError (bad sizes / pointers) */
  TSQ_ERR_BUSY = 6,               /* -> RuntimeError("not reentrant") */
  TSQ_ERR_CAPACITY = 7            /* internal queue overflow (cannot happen: the queues
                                   * are drained before they could overflow) */
} tsq_status;

/* One stage of a host-driven level, reported to the on_level callback (the
 * stage_hook(a, b, new_l, new_r, pivot) / trace STAGE_END contract,
 * core.py:1705-1710): inclusive bounds a..b, keys[a..new_l] < pivot,
 * keys[new_l+1..new_r-1] == pivot, keys[new_r..b] > pivot. */
typedef enum {
  TSQ_STAGE_PARTITION = 0,        /* three-way partition pass (_run_machine) */
  TSQ_STAGE_SORTED = 1,           /* verified sorted, bypassed (_sorted_handler) */
  TSQ_STAGE_REVERSED = 2,         /* verified reversed, mirrored (_reversed_handler) */
  TSQ_STAGE_HANDLER_FALLBACK = 3  /* verification failed: partitioned next level;
                                   * new_l = the handler tried (TSQ_STAGE_SORTED or
                                   * TSQ_STAGE_REVERSED), new_r unset */
} tsq_stage_kind;

typedef struct {
  int64_t a, b, new_l, new_r;
  uint64_t pivot;                 /* raw bits of a key of key_t */
  int32_t kind;                   /* tsq_stage_kind */
  int32_t depth;                  /* recursion depth of the stage (root = 1) */
} tsq_stage_record;

/* Called after every host-driven level once the caller's keys/payload hold
 * each listed segment's post-stage contents (in stage-export mode the sort
 * runs in an internal copy and the caller's buffers are a view of the
 * recursion; they receive the sorted result at the end). */
typedef void (*tsq_level_fn)(void *user, int32_t level, const tsq_stage_record *records,
                             uint32_t count);

typedef enum {
  TSQ_NONE = 0,
  TSQ_I32 = 1,
  TSQ_U32 = 2,
  TSQ_I64 = 3,
  TSQ_U64 = 4,
  TSQ_F32 = 5,
  TSQ_F64 = 6
} tsq_dtype;

/* GPU knobs (kept apart from SortConfig, whose validation caps
 * insertion_threshold below 70, config.py:31-38). 0 = default. */
typedef struct {
  double dran;             /* MitigationRng.dran in [0.5,1.5) (pivot.py:45-49); 0 -> 1.0 */
  int32_t mitigation;      /* jitter sample positions by dran (config.py:24) */
  int32_t fast_paths;      /* sorted/reversed verify-and-bypass (core.py:1678-1698); default 1 */
  int32_t max_depth;       /* depth guard: deeper segments are split at the midpoint of
                            * their key bounds (no sampling), which ends the recursion
                            * within key-bits more levels; 0 = max(24, 2 log2 n) */
  int32_t host_levels;     /* 1 = drive levels from the host (debug/per-level stats) */
  int32_t small_threshold; /* segments <= this go on chip (1..40952); 0 = the default:
                            * bare 4-byte keys 40952, bare 8-byte keys 16376, records
                            * 8184; clamped to the key type's on-chip capacity */
  int32_t reproducible;    /* 1 = run-to-run identical layout (decoupled look-back);
                            * 0 = tiles reserve output ranges with one atomic (faster) */
  int32_t stage_export;    /* 1 = host-driven levels with on_level called per level */
  tsq_level_fn on_level;   /* stage_export callback (may be NULL) */
  void *on_level_user;
  int64_t reserved[1];
} tsq_params;

/* Counters of one call (the SortStats analogue, stats.py:33-70). */
typedef struct {
  uint64_t n;
  uint64_t stages;             /* segments partitioned or verified on device */
  uint64_t levels;             /* device partition levels (HBM passes) */
  uint64_t max_depth;          /* deepest recursion level reached */
  uint64_t small_segments;     /* segments finished by the on-chip sort */
  uint64_t eq_runs;            /* ==p runs retired */
  uint64_t eq_elements;        /* keys retired inside ==p runs */
  uint64_t sorted_bypass;      /* stages verified sorted (no migration) */
  uint64_t reversed_bypass;    /* stages verified reversed (mirrored) */
  uint64_t verify_fallbacks;   /* verification failed -> partitioned */
  uint64_t partitioned_elements;
  uint64_t bytes_partition;    /* algorithmic HBM bytes of the level kernels */
  uint64_t bytes_small;        /* ... of the on-chip sort */
  uint64_t bytes_retire;       /* ... of run retirement (fills / copies) */
  uint64_t temp_high_water;    /* workspace elements reserved */
  uint64_t error_flags;
  uint64_t writes_caller;      /* element writes into the caller's array */
  uint64_t writes_workspace;   /* element writes into the workspace */
  uint64_t bisected;           /* segments split at their key-bound midpoint (depth guard) */
  uint64_t flushes;            /* mid-recursion drains of the on-chip / run queues */
  float ms_levels;             /* device time of the level loop (events) */
  float ms_total;              /* device time of the whole sort (events) */
} tsq_stats;

typedef struct tsq_workspace tsq_workspace;

const char *tsq_status_str(tsq_status s);
int tsq_abi_version(void);

/* Workspace lifecycle (TempStore, core.py:81-104). */
tsq_status tsq_workspace_create(tsq_workspace **out, int device);
void tsq_workspace_destroy(tsq_workspace *ws);
/* bytes of device memory a sort of n elements needs */
size_t tsq_workspace_bytes(size_t n, tsq_dtype key_t, tsq_dtype payload_t);
/* reserve for n elements; keeps the high water (no shrink) */
tsq_status tsq_workspace_reserve(tsq_workspace *ws, size_t n, tsq_dtype key_t,
                                 tsq_dtype payload_t);
/* release device memory; the next sort reallocates (free_temp_storage) */
tsq_status tsq_workspace_free(tsq_workspace *ws);
/* elements the workspace currently holds capacity for; allocation count */
size_t tsq_workspace_capacity(const tsq_workspace *ws);
uint64_t tsq_workspace_alloc_count(const tsq_workspace *ws);
/* Outcome of the last sort on this workspace: waits for it (on `stream`)
 * and maps its device error flags to a status (TSQ_OK when it finished). */
tsq_status tsq_workspace_last_status(tsq_workspace *ws, void *stream);

/* Sort keys[0..n) ascending in place; payload (nullable, TSQ_U32) moves with
 * its key (records compared by key only).  keys must be aligned to its
 * element size and payload to 4 bytes (else TSQ_ERR_INVALID); buffers that
 * are not 16-byte aligned (views with a storage offset) are sorted through
 * an aligned workspace copy.  stats may be NULL: the call then returns
 * without synchronising, and tsq_workspace_last_status reports the
 * outcome. */
tsq_status tsq_sort(void *keys, void *payload, size_t n, tsq_dtype key_t,
                    tsq_dtype payload_t, const tsq_params *params,
                    tsq_workspace *ws, void *stream, tsq_stats *stats);

/* Per-level trace of the last host_levels sort (the stage_hook / trace
 * analogue, core.py:1705-1710): device ms of the partition pass and of the
 * scheduling pass, live segments, tiles and algorithmic HBM bytes of the
 * partition pass per level.  Returns the number of levels (may exceed cap);
 * any output pointer may be NULL. */
int tsq_level_trace(const tsq_workspace *ws, float *part_ms, float *sched_ms,
                    uint32_t *segments, uint32_t *tiles, uint64_t *bytes, int cap);

/* One stage: three-way partition of keys[0..n) around `pivot` (raw bits of a
 * key of key_t), out of place into out_keys (and out_payload), < from the
 * front, > from the back, == in the middle.  Writes new_l = n_lt - 1 and
 * new_r = n - n_gt (stage law, reference tests/conftest.py:37-45). Syncs. */
tsq_status tsq_partition_segment(const void *keys, const void *payload,
                                 void *out_keys, void *out_payload, size_t n,
                                 tsq_dtype key_t, tsq_dtype payload_t,
                                 uint64_t pivot, tsq_workspace *ws,
                                 void *stream, int64_t *new_l, int64_t *new_r);

/* Device pivot sampling of keys[0..n): writes the chosen pivot (raw bits)
 * and the sample order flag (+1 nondecreasing, -1 nonincreasing, 0).  Syncs. */
tsq_status tsq_select_pivot(const void *keys, size_t n, tsq_dtype key_t,
                            double dran, int32_t mitigation,
                            tsq_workspace *ws, void *stream,
                            uint64_t *pivot, int32_t *order_flag);

/* Late swapping (bigelem.py:31-99): dst_rows[i] = src_rows[perm[i]] for n
 * rows of row_bytes each (device pointers, distinct buffers; perm a device
 * array of n uint32 origins, i.e. the payload of a (key, index) records
 * sort).  Enqueued on `stream`, does not sync. */
tsq_status tsq_apply_permutation(const void *src_rows, void *dst_rows, size_t n,
                                 size_t row_bytes, const uint32_t *perm, void *stream);

#ifdef __cplusplus
}
#endif
#endif
