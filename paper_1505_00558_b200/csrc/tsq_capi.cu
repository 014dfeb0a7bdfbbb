// tsq_capi.cu -- host side of libtsq_b200.so: workspace (the retained
// TempStore analogue, core.py:81-104), the CUDA-graph driver of the device
// recursion (Sorter._range, core.py:1643-1728, with no per-level host round
// trip: a conditional WHILE node re-launches the level kernel until the
// device queue is empty), and the extern "C" entry points of include/tsq.h.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "tsq_kernels.cuh"

using namespace tsq;

namespace {

struct KernelSet {
  const void *init, *part, *sched, *retire, *selp, *exportk;
  int key_bytes, tile;
  size_t part_smem, sched_smem;
  // on-chip sort classes: 256 / 512 threads (tsq_small.cuh)
  const void *small[kSmallClasses];
  size_t small_smem[kSmallClasses];
  int small_threads[kSmallClasses];
  int small_cap[kSmallClasses];  // keys each class takes
  bool raw_order;  // the workspace buffer keeps the caller's encoding too
};

int key_bytes_of(int dt);

// Default on-chip cut (measured on B200, scripts/cut_sweep.py, profiles/r02*):
// bare 4-byte keys 40952 = the largest class (uniform int32 2^26: 1.87 ms
// against 1.94 at 32760; 2^24: 0.64 / 0.68 / 0.72 at 16376; 2^20: 0.208 /
// 0.208 / 0.222 / 0.230 at 8184) -- a radix pass over one more key bit costs
// less than the partition level it saves, at every size.  Bare 8-byte keys
// 16376, their largest class too (normal f64 2^26: 3.67 ms against 3.98 at
// 8184).  Records 8184: their largest class runs 1024 threads at one CTA
// per SM (records 2^27: 9.79 ms at 8192, 9.90 at 16384).
// (A class of S item slots takes segments of <= S - kSmallSlack keys.)
int default_small_t(int kt, int pt, size_t n) {
  (void)n;
  const bool pay = pt == TSQ_U32;
  if (!pay) return (key_bytes_of(kt) == 4 ? kSmallGiant : kSmallHuge) - kSmallSlack;
  return kSmallMax - kSmallSlack;
}

template <int DT, bool PAY>
KernelSet make_set() {
  typedef Codec<DT> C;
  typedef typename C::U U;
  KernelSet s;
  s.init = reinterpret_cast<const void *>(&init_kernel<C, PAY>);
  s.part = reinterpret_cast<const void *>(&partition_kernel<C, PAY>);
  s.sched = reinterpret_cast<const void *>(&schedule_kernel<C, PAY>);
  s.small[0] = reinterpret_cast<const void *>(&small_sort_kernel<C, PAY, 0>);
  s.small[1] = reinterpret_cast<const void *>(&small_sort_kernel<C, PAY, 1>);
  s.small[2] = reinterpret_cast<const void *>(&small_sort_kernel<C, PAY, 2>);
  s.small_smem[0] = RadixGeo<C, PAY, 0>::SMEM;
  s.small_smem[1] = RadixGeo<C, PAY, 1>::SMEM;
  s.small_smem[2] = RadixGeo<C, PAY, 2>::SMEM;
  s.small_threads[0] = RadixGeo<C, PAY, 0>::NT;
  s.small_threads[1] = RadixGeo<C, PAY, 1>::NT;
  s.small_threads[2] = RadixGeo<C, PAY, 2>::NT;
  s.small_cap[0] = RadixGeo<C, PAY, 0>::CAP;
  s.small_cap[1] = RadixGeo<C, PAY, 1>::CAP;
  s.small_cap[2] = RadixGeo<C, PAY, 2>::CAP;
  s.raw_order = C::kRawOrder;
  s.retire = reinterpret_cast<const void *>(&retire_kernel<C, PAY>);
  s.selp = reinterpret_cast<const void *>(&select_pivot_kernel<C>);
  s.exportk = reinterpret_cast<const void *>(&export_level_kernel<C, PAY>);
  s.key_bytes = (int)sizeof(U);
  s.tile = Geo<C, PAY>::TILE;
  s.part_smem = Geo<C, PAY>::SMEM;
  s.sched_smem = (size_t)(kThreads / 32) * (kMaxSample + 1) * sizeof(U);
  return s;
}

bool get_set(int dt, bool pay, KernelSet *out) {
#define TSQ_CASE(D)                                          \
  case D:                                                    \
    *out = pay ? make_set<D, true>() : make_set<D, false>(); \
    return true;
#ifdef TSQ_ONLY  // experiment builds (scripts/variants.py): one (dtype, payload) set only
  if (dt * 2 + (pay ? 1 : 0) != TSQ_ONLY) return false;
  *out = make_set<TSQ_ONLY / 2, (TSQ_ONLY & 1) != 0>();
  return true;
#else
  switch (dt) {
    TSQ_CASE(TSQ_I32)
    TSQ_CASE(TSQ_U32)
    TSQ_CASE(TSQ_F32)
    TSQ_CASE(TSQ_I64)
    TSQ_CASE(TSQ_U64)
    TSQ_CASE(TSQ_F64)
    default:
      return false;
  }
#endif
#undef TSQ_CASE
}

int key_bytes_of(int dt) {
  switch (dt) {
    case TSQ_I32: case TSQ_U32: case TSQ_F32: return 4;
    case TSQ_I64: case TSQ_U64: case TSQ_F64: return 8;
    default: return 0;
  }
}

// host copies of the order-preserving codecs (for given pivots)
u64 host_enc(int dt, u64 x) {
  switch (dt) {
    case TSQ_I32: return (x ^ 0x80000000ull) & 0xffffffffull;
    case TSQ_U32: return x & 0xffffffffull;
    case TSQ_F32: { uint32_t v = (uint32_t)x; return (u64)(v ^ ((0u - (v >> 31)) | 0x80000000u)); }
    case TSQ_I64: return x ^ 0x8000000000000000ull;
    case TSQ_U64: return x;
    case TSQ_F64: return x ^ ((0ull - (x >> 63)) | 0x8000000000000000ull);
    default: return x;
  }
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t keys_alt, pay_alt, side_pay, segs[2], tilemap[2], lookback[2], sq[kSmallClasses], runs,
      chunkmap;
  size_t stage_keys, stage_pay;  // aligned copies of the caller's buffers (staged sorts)
  size_t stage_out;              // per-segment stage records (stage-export mode)
  size_t total;
  uint32_t seg_cap, tile_cap, run_cap, chunk_cap, sq_cap[kSmallClasses];
};

Layout make_layout(size_t n, int kt, int pt, int small_t = 0, bool staged = false,
                   bool export_records = false) {
  if (small_t <= 0) small_t = default_small_t(kt, pt, n);
  Layout L;
  memset(&L, 0, sizeof(L));
  const int kb = key_bytes_of(kt);
  const size_t tile = kb == 4 ? 4096 : 2048;
  const bool pay = pt == TSQ_U32;
  L.seg_cap = (uint32_t)(n / (size_t)small_t + 2);
  L.tile_cap = (uint32_t)(n / tile + 2ull * L.seg_cap + 2);
  L.run_cap = 8u * L.seg_cap + 64u;
  L.sq_cap[0] = 2u * L.run_cap;
  L.sq_cap[1] = (uint32_t)(n / (size_t)(kSmallT - kSmallSlack + 1) + 2);
  L.sq_cap[2] = (uint32_t)(n / (size_t)(kSmallMax - kSmallSlack + 1) + 2);
  if (getenv("TSQ_DEBUG_MIN_QUEUES")) {
    // test knob: the smallest queues the flush rule allows, so the level
    // loop drains them every level or two (exercises the drain rounds)
    L.run_cap = L.seg_cap + 64u;
    L.sq_cap[0] = 2u * L.seg_cap + 64u;
  }
  L.chunk_cap = (uint32_t)(n / kRunChunk + L.run_cap + 2);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.keys_alt = take(n * kb + 64);
  L.pay_alt = take(pay ? n * 4 + 64 : 0);
  L.side_pay = take(pay ? n * 4 + 64 : 0);
  for (int b = 0; b < 2; ++b) L.segs[b] = take((size_t)L.seg_cap * sizeof(Seg));
  for (int b = 0; b < 2; ++b) L.tilemap[b] = take((size_t)L.tile_cap * 4);
  for (int b = 0; b < 2; ++b) L.lookback[b] = take((size_t)L.tile_cap * 8);
  for (int c = 0; c < kSmallClasses; ++c) L.sq[c] = take((size_t)L.sq_cap[c] * sizeof(SmallSeg));
  L.runs = take((size_t)L.run_cap * sizeof(Run));
  L.chunkmap = take((size_t)L.chunk_cap * 4);
  // a caller buffer that is element- but not 16-byte-aligned (a CUDA view
  // with a storage offset, e.g. x[1:]) is sorted in an aligned copy: the
  // partition pass writes whole runs with cp.async.bulk, which needs
  // 16-byte-aligned global addresses
  L.stage_keys = take(staged ? n * kb + 64 : 0);
  L.stage_pay = take(staged && pay ? n * 4 + 64 : 0);
  L.stage_out = take(export_records ? (size_t)L.seg_cap * sizeof(StageRecord) : 0);
  L.total = off;
  return L;
}

struct GraphEntry {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t init_node = nullptr;
  cudaGraphConditionalHandle cond = 0, cond_outer = 0;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  cudaKernelNodeParams init_params;
};

static_assert(sizeof(StageRecord) == sizeof(tsq_stage_record), "stage record layout");
static_assert(sizeof(tsq_params) == 64, "tsq_params layout (tests/test_api_cpu.py)");
static_assert(sizeof(tsq_stats) == 168, "tsq_stats layout (tests/test_api_cpu.py)");

}  // namespace

struct tsq_workspace {
  int device = 0;
  int num_sms = 148;
  void *block = nullptr;
  size_t block_bytes = 0;
  size_t cap_elems = 0;
  uint64_t alloc_count = 0;
  Params *d_params = nullptr;
  Ctl *d_ctl = nullptr;
  Ctl *h_ctl_dev = nullptr;  // device alias of the mapped host copy h_ctl
  Ctl *h_ctl = nullptr;
  cudaEvent_t done = nullptr;
  bool active = false;
  std::mutex mu;
  std::map<int, GraphEntry> graphs;
  std::vector<float> level_ms, sched_ms;  // host_levels mode trace
  std::vector<uint64_t> level_bytes;
  std::vector<uint32_t> level_segs, level_tiles;
  std::vector<tsq_stage_record> records;  // stage-export mode, one level
};

#define TSQ_CUDA(call)                                     \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) {                               \
      fprintf(stderr, "tsq: %s failed: %s (%s:%d)\n", #call, \
              cudaGetErrorString(e_), __FILE__, __LINE__); \
      return TSQ_ERR_CUDA;                                 \
    }                                                      \
  } while (0)

namespace {

// Every entry point runs on the workspace's device and leaves the caller's
// current device as it found it.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int occupancy_grid(tsq_workspace *ws, const void *fn, size_t smem, int block = kThreads) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem) != cudaSuccess ||
      occ < 1)
    occ = 1;
  return occ * ws->num_sms;
}

tsq_status prepare_small_smem(const KernelSet &ks) {
  const void *fns[2 + kSmallClasses] = {ks.part, ks.sched, ks.small[0], ks.small[1], ks.small[2]};
  const size_t sm[2 + kSmallClasses] = {ks.part_smem, ks.sched_smem, ks.small_smem[0],
                                        ks.small_smem[1], ks.small_smem[2]};
  // always opt in: dynamic + static shared memory may cross 48 KB even when
  // the dynamic part alone does not
  for (int i = 0; i < 2 + kSmallClasses; ++i)
    if (fns[i]) TSQ_CUDA(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm[i]));
  return TSQ_OK;
}

// one recursion level = partition pass + segment scheduling
struct LevelLaunch {
  dim3 part_grid, sched_grid;
};

LevelLaunch level_launch(tsq_workspace *ws, const KernelSet &ks) {
  LevelLaunch L;
  L.part_grid = dim3(occupancy_grid(ws, ks.part, ks.part_smem, kPartThreads));
#ifdef TSQ_SCHED_PER_SM
  L.sched_grid = dim3(TSQ_SCHED_PER_SM * ws->num_sms);
#else
  L.sched_grid = dim3(occupancy_grid(ws, ks.sched, ks.sched_smem));
#endif
  return L;
}

// (the partition and schedule kernels also take the control block's address
// by value -- it never moves for a workspace -- so their first read of it does
// not wait for the read of the parameter block)
cudaError_t launch_level(const KernelSet &ks, const LevelLaunch &L, Params **dst, Ctl **ctl,
                         cudaStream_t s) {
  void *args[2] = {dst, ctl};
  cudaError_t e = cudaLaunchKernel(ks.part, L.part_grid, dim3(kPartThreads), args, ks.part_smem, s);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernel(ks.sched, L.sched_grid, dim3(kThreads), args, ks.sched_smem, s);
}

// the on-chip sort classes, retirement and the queue reset (a drain round)
cudaError_t launch_drain(tsq_workspace *ws, const KernelSet &ks, Params **dst, cudaStream_t s) {
  void *args[1] = {dst};
  for (int c = 0; c < kSmallClasses; ++c) {
    if (!ks.small[c]) continue;
    cudaError_t e = cudaLaunchKernel(
        ks.small[c], dim3(occupancy_grid(ws, ks.small[c], ks.small_smem[c], ks.small_threads[c])),
        dim3(ks.small_threads[c]), args, ks.small_smem[c], s);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaLaunchKernel(ks.retire, dim3(occupancy_grid(ws, ks.retire, 0)),
                                   dim3(kThreads), args, 0, s);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernel(reinterpret_cast<const void *>(&drain_kernel), dim3(1), dim3(32), args,
                          0, s);
}

void fill_params(tsq_workspace *ws, const Layout &L, Params *p, void *keys, void *payload,
                 size_t n) {
  memset(p, 0, sizeof(*p));
  char *base = reinterpret_cast<char *>(ws->block);
  p->keys[0] = keys;
  p->keys[1] = base + L.keys_alt;
  p->pay[0] = reinterpret_cast<uint32_t *>(payload);
  p->pay[1] = payload ? reinterpret_cast<uint32_t *>(base + L.pay_alt) : nullptr;
  p->side_pay = payload ? reinterpret_cast<uint32_t *>(base + L.side_pay) : nullptr;
  p->n = (long long)n;
  p->raw[0] = 1;
  p->raw[1] = 0;
  const bool a0 = ((uintptr_t)keys % 16 == 0) && ((uintptr_t)payload % 16 == 0);
  p->aligned[0] = a0 ? 1 : 0;
  p->aligned[1] = 1;
  for (int b = 0; b < 2; ++b) {
    p->segs[b] = reinterpret_cast<Seg *>(base + L.segs[b]);
    p->tilemap[b] = reinterpret_cast<uint32_t *>(base + L.tilemap[b]);
    p->lookback[b] = reinterpret_cast<u64 *>(base + L.lookback[b]);
  }
  for (int c = 0; c < kSmallClasses; ++c) {
    p->sq[c] = reinterpret_cast<SmallSeg *>(base + L.sq[c]);
    p->sq_cap[c] = L.sq_cap[c];
  }
  p->runs = reinterpret_cast<Run *>(base + L.runs);
  p->chunkmap = reinterpret_cast<uint32_t *>(base + L.chunkmap);
  p->seg_cap = L.seg_cap;
  p->tile_cap = L.tile_cap;
  p->run_cap = L.run_cap;
  p->chunk_cap = L.chunk_cap;
  p->ctl = ws->d_ctl;
  p->max_depth = 96;
  p->fast_paths = 1;
  p->mitigation = 1;
  p->dran = 1.0;
  p->small_t = kSmallMax - kSmallSlack;
  p->sq_lim[0] = kSmallT - kSmallSlack;
  p->sq_lim[1] = kSmallMax - kSmallSlack;
  p->sq_lim[2] = kSmallMax - kSmallSlack;
  p->reproducible = 0;
}

// The whole sort as one graph, no host round trip per level:
//   init -> WHILE(outer) { WHILE(inner) { partition -> schedule }
//                          -> small sorts || retire -> drain }
// The last schedule CTA of a level keeps the inner loop going while
// segments remain; when the on-chip or run queues could not take another
// level it ends the inner loop early (a flush), the drain round empties
// them and the outer loop re-enters the level loop.  Normally the outer
// body runs once.
tsq_status build_graph(tsq_workspace *ws, int kt, bool pay, GraphEntry *ge) {
  KernelSet ks;
  if (!get_set(kt, pay, &ks)) return TSQ_ERR_UNSUPPORTED_DTYPE;
  tsq_status st = prepare_small_smem(ks);
  if (st != TSQ_OK) return st;
  for (int i = 0; i < 3; ++i) TSQ_CUDA(cudaEventCreate(&ge->ev[i]));
  TSQ_CUDA(cudaGraphCreate(&ge->graph, 0));
  cudaGraph_t g = ge->graph;
  cudaGraphNode_t e0, e1, e2, onode, inode, lnode, schednode;
  TSQ_CUDA(cudaGraphAddEventRecordNode(&e0, g, nullptr, 0, ge->ev[0]));

  static Params dummy;  // replaced per call via cudaGraphExecKernelNodeSetParams
  memset(&dummy, 0, sizeof(dummy));
  static Params *dummy_dst = nullptr;
  dummy_dst = ws->d_params;
  ge->init_params = cudaKernelNodeParams{};
  void *init_args[2] = {&dummy, &dummy_dst};
  ge->init_params.func = const_cast<void *>(ks.init);
  ge->init_params.gridDim = dim3(1);
  ge->init_params.blockDim = dim3(kThreads);
  ge->init_params.sharedMemBytes = 0;
  ge->init_params.kernelParams = init_args;
  TSQ_CUDA(cudaGraphAddKernelNode(&ge->init_node, g, &e0, 1, &ge->init_params));
  TSQ_CUDA(cudaGraphAddEventRecordNode(&e1, g, &ge->init_node, 1, ge->ev[1]));

  // both handles live in the top-level graph: the outer one enters its body
  // once per launch by default; the init kernel sets the inner one
  TSQ_CUDA(cudaGraphConditionalHandleCreate(&ge->cond_outer, g, 1, cudaGraphCondAssignDefault));
  TSQ_CUDA(cudaGraphConditionalHandleCreate(&ge->cond, g, 0, 0));
  // cudaGraphNodeParams has a deleted default constructor (union member)
  alignas(cudaGraphNodeParams) unsigned char op_raw[sizeof(cudaGraphNodeParams)];
  memset(op_raw, 0, sizeof(op_raw));
  cudaGraphNodeParams &op = *reinterpret_cast<cudaGraphNodeParams *>(op_raw);
  op.type = cudaGraphNodeTypeConditional;
  op.conditional.handle = ge->cond_outer;
  op.conditional.type = cudaGraphCondTypeWhile;
  op.conditional.size = 1;
  TSQ_CUDA(cudaGraphAddNode(&onode, g, &e1, 1, &op));
  cudaGraph_t obody = op.conditional.phGraph_out[0];

  alignas(cudaGraphNodeParams) unsigned char ip_raw[sizeof(cudaGraphNodeParams)];
  memset(ip_raw, 0, sizeof(ip_raw));
  cudaGraphNodeParams &ip = *reinterpret_cast<cudaGraphNodeParams *>(ip_raw);
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = ge->cond;
  ip.conditional.type = cudaGraphCondTypeWhile;
  ip.conditional.size = 1;
  TSQ_CUDA(cudaGraphAddNode(&inode, obody, nullptr, 0, &ip));
  cudaGraph_t body = ip.conditional.phGraph_out[0];

  Params *dp = ws->d_params;
  Ctl *dctl = ws->d_ctl;
  void *dev_args[2] = {&dp, &dctl};
  const LevelLaunch LL = level_launch(ws, ks);
  cudaKernelNodeParams pk = cudaKernelNodeParams{};
  pk.func = const_cast<void *>(ks.part);
  pk.gridDim = LL.part_grid;
  pk.blockDim = dim3(kPartThreads);
  pk.sharedMemBytes = (unsigned)ks.part_smem;
  pk.kernelParams = dev_args;
  TSQ_CUDA(cudaGraphAddKernelNode(&lnode, body, nullptr, 0, &pk));
  cudaKernelNodeParams lk = cudaKernelNodeParams{};
  lk.func = const_cast<void *>(ks.sched);
  lk.gridDim = LL.sched_grid;
  lk.blockDim = dim3(kThreads);
  lk.sharedMemBytes = (unsigned)ks.sched_smem;
  lk.kernelParams = dev_args;
  TSQ_CUDA(cudaGraphAddKernelNode(&schednode, body, &lnode, 1, &lk));

  cudaGraphNode_t tail[kSmallClasses + 1];
  int ntail = 0;
  for (int c = 0; c < kSmallClasses; ++c) {
    if (!ks.small[c]) continue;
    cudaKernelNodeParams sk = lk;
    sk.func = const_cast<void *>(ks.small[c]);
    sk.gridDim = dim3(occupancy_grid(ws, ks.small[c], ks.small_smem[c], ks.small_threads[c]));
    sk.blockDim = dim3(ks.small_threads[c]);
    sk.sharedMemBytes = (unsigned)ks.small_smem[c];
    TSQ_CUDA(cudaGraphAddKernelNode(&tail[ntail++], obody, &inode, 1, &sk));
  }
  cudaKernelNodeParams rk = lk;
  rk.func = const_cast<void *>(ks.retire);
  rk.gridDim = dim3(occupancy_grid(ws, ks.retire, 0));
  rk.sharedMemBytes = 0;
  TSQ_CUDA(cudaGraphAddKernelNode(&tail[ntail++], obody, &inode, 1, &rk));
  cudaKernelNodeParams dk = lk;
  dk.func = reinterpret_cast<void *>(&drain_kernel);
  dk.gridDim = dim3(1);
  dk.blockDim = dim3(32);
  dk.sharedMemBytes = 0;
  cudaGraphNode_t dnode;
  TSQ_CUDA(cudaGraphAddKernelNode(&dnode, obody, tail, ntail, &dk));
  TSQ_CUDA(cudaGraphAddEventRecordNode(&e2, g, &onode, 1, ge->ev[2]));
  TSQ_CUDA(cudaGraphInstantiate(&ge->exec, g, 0));
  return TSQ_OK;
}

tsq_status reserve_locked(tsq_workspace *ws, size_t n, int kt, int pt, int small_t = 0,
                          bool staged = false, bool export_records = false) {
  const Layout L = make_layout(n, kt, pt, small_t, staged, export_records);
  if (L.total <= ws->block_bytes) {
    if (n > ws->cap_elems) ws->cap_elems = n;
    return TSQ_OK;
  }
  if (ws->block) {
    cudaEventSynchronize(ws->done);
    cudaFree(ws->block);
    ws->block = nullptr;
    ws->block_bytes = 0;
    ws->cap_elems = 0;
  }
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, L.total);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return TSQ_ERR_ALLOC;
  }
  ws->block = p;
  ws->block_bytes = L.total;
  ws->cap_elems = n;
  ws->alloc_count += 1;
  return TSQ_OK;
}

tsq_status check_args(size_t n, int kt, int pt) {
  if (key_bytes_of(kt) == 0) return TSQ_ERR_UNSUPPORTED_DTYPE;
  if (pt != TSQ_NONE && pt != TSQ_U32) return TSQ_ERR_UNSUPPORTED_DTYPE;
  if (n >= (1ull << 31)) return TSQ_ERR_INVALID;
  return TSQ_OK;
}

// element alignment of a caller buffer is required; 16-byte alignment is
// not (a misaligned buffer is sorted through an aligned copy)
bool element_aligned(const void *p, size_t bytes) { return p == nullptr || (uintptr_t)p % bytes == 0; }
bool bulk_aligned(const void *p) { return p == nullptr || (uintptr_t)p % 16 == 0; }

// The control block comes back through mapped host memory written by a tiny
// kernel, not a memcpy: a copy would queue on the copy engine behind any
// large device->host transfer in flight on other streams (sort_many's
// pipeline), stalling the host for that transfer's duration.
tsq_status read_ctl(tsq_workspace *ws, cudaStream_t s) {
  void *args[2] = {&ws->d_ctl, &ws->h_ctl_dev};
  TSQ_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(&publish_ctl_kernel), dim3(1),
                            dim3(32), args, 0, s));
  TSQ_CUDA(cudaStreamSynchronize(s));
  return TSQ_OK;
}

tsq_status status_of(uint32_t error) {
  if (error & (ERR_DEPTH | ERR_LEVELS)) return TSQ_ERR_DEPTH_EXCEEDED;
  if (error) return TSQ_ERR_CAPACITY;
  return TSQ_OK;
}

tsq_status fill_stats(tsq_workspace *ws, size_t n, tsq_stats *st) {
  const Ctl &c = *ws->h_ctl;
  memset(st, 0, sizeof(*st));
  st->n = n;
  st->stages = c.stages;
  st->levels = c.levels;
  st->max_depth = c.max_depth;
  st->small_segments = c.small_segs_done;
  for (int q = 0; q < kSmallClasses; ++q) st->small_segments += c.sq_count[q];
  st->eq_runs = c.eq_runs;
  st->eq_elements = c.eq_elements;
  st->sorted_bypass = c.sorted_bypass;
  st->reversed_bypass = c.reversed_bypass;
  st->verify_fallbacks = c.verify_fallbacks;
  st->partitioned_elements = c.partitioned_elements;
  st->bytes_partition = c.bytes_partition;
  st->bytes_small = c.bytes_small;
  st->bytes_retire = c.bytes_retire;
  st->temp_high_water = ws->cap_elems;
  st->error_flags = c.error;
  st->writes_caller = c.writes0;
  st->writes_workspace = c.writes1;
  st->bisected = c.bisected;
  st->flushes = c.flushes;
  return status_of(c.error);
}

struct ActiveGuard {
  tsq_workspace *ws;
  explicit ActiveGuard(tsq_workspace *w) : ws(w) {}
  ~ActiveGuard() {
    std::lock_guard<std::mutex> lk(ws->mu);
    ws->active = false;
  }
};

tsq_status acquire(tsq_workspace *ws) {
  std::lock_guard<std::mutex> lk(ws->mu);
  if (ws->active) return TSQ_ERR_BUSY;
  ws->active = true;
  return TSQ_OK;
}

struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// default depth guard: max(24, 2 * ceil(log2 n)) levels of sampled pivots
int default_max_depth(size_t n) {
  int lg = 0;
  while (lg < 63 && (1ull << lg) < n) ++lg;
  return 2 * lg > 24 ? 2 * lg : 24;
}

}  // namespace

extern "C" {

const char *tsq_status_str(tsq_status s) {
  switch (s) {
    case TSQ_OK: return "ok";
    case TSQ_ERR_ALLOC: return "device workspace allocation failed";
    case TSQ_ERR_UNSUPPORTED_DTYPE: return "unsupported dtype";
    case TSQ_ERR_CUDA: return "CUDA error";
    case TSQ_ERR_DEPTH_EXCEEDED: return "recursion level limit reached";
    case TSQ_ERR_INVALID: return "invalid argument";
    case TSQ_ERR_BUSY: return "sorter instance is not reentrant";
    case TSQ_ERR_CAPACITY: return "device queue capacity exceeded";
  }
  return "unknown status";
}

int tsq_abi_version(void) { return TSQ_ABI_VERSION; }

tsq_status tsq_workspace_create(tsq_workspace **out, int device) {
  if (!out) return TSQ_ERR_INVALID;
  *out = nullptr;
  DeviceGuard dg(device);
  if (!dg.ok) return TSQ_ERR_CUDA;
  tsq_workspace *ws = new tsq_workspace();
  ws->device = device;
  cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&ws->d_params, sizeof(Params)) != cudaSuccess ||
      cudaMalloc(&ws->d_ctl, sizeof(Ctl)) != cudaSuccess ||
      cudaHostAlloc(&ws->h_ctl, sizeof(Ctl), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&ws->h_ctl_dev, ws->h_ctl, 0) != cudaSuccess) {
    cudaGetLastError();
    tsq_workspace_destroy(ws);
    return TSQ_ERR_ALLOC;
  }
  memset(ws->h_ctl, 0, sizeof(Ctl));
  cudaMemset(ws->d_ctl, 0, sizeof(Ctl));
  TSQ_CUDA(cudaEventCreateWithFlags(&ws->done, cudaEventDisableTiming));
  *out = ws;
  return TSQ_OK;
}

void tsq_workspace_destroy(tsq_workspace *ws) {
  if (!ws) return;
  DeviceGuard dg(ws->device);
  if (ws->done) cudaEventSynchronize(ws->done);
  for (auto &kv : ws->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
    for (auto e : kv.second.ev)
      if (e) cudaEventDestroy(e);
  }
  if (ws->block) cudaFree(ws->block);
  if (ws->d_params) cudaFree(ws->d_params);
  if (ws->d_ctl) cudaFree(ws->d_ctl);
  if (ws->h_ctl) cudaFreeHost(ws->h_ctl);
  if (ws->done) cudaEventDestroy(ws->done);
  delete ws;
}

size_t tsq_workspace_bytes(size_t n, tsq_dtype key_t, tsq_dtype payload_t) {
  if (check_args(n, key_t, payload_t) != TSQ_OK) return 0;
  return make_layout(n, key_t, payload_t).total;
}

tsq_status tsq_workspace_reserve(tsq_workspace *ws, size_t n, tsq_dtype key_t,
                                 tsq_dtype payload_t) {
  if (!ws) return TSQ_ERR_INVALID;
  tsq_status st = check_args(n, key_t, payload_t);
  if (st != TSQ_OK) return st;
  st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard g(ws);
  DeviceGuard dg(ws->device);
  return reserve_locked(ws, n, key_t, payload_t);
}

tsq_status tsq_workspace_free(tsq_workspace *ws) {
  if (!ws) return TSQ_ERR_INVALID;
  tsq_status st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard g(ws);
  DeviceGuard dg(ws->device);
  if (ws->block) {
    cudaEventSynchronize(ws->done);
    cudaFree(ws->block);
  }
  ws->block = nullptr;
  ws->block_bytes = 0;
  ws->cap_elems = 0;
  return TSQ_OK;
}

size_t tsq_workspace_capacity(const tsq_workspace *ws) { return ws ? ws->cap_elems : 0; }
uint64_t tsq_workspace_alloc_count(const tsq_workspace *ws) { return ws ? ws->alloc_count : 0; }

tsq_status tsq_workspace_last_status(tsq_workspace *ws, void *stream) {
  if (!ws) return TSQ_ERR_INVALID;
  tsq_status st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard g(ws);
  DeviceGuard dg(ws->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TSQ_CUDA(cudaStreamWaitEvent(s, ws->done, 0));
  st = read_ctl(ws, s);
  if (st != TSQ_OK) return st;
  return status_of(ws->h_ctl->error);
}

tsq_status tsq_sort(void *keys, void *payload, size_t n, tsq_dtype key_t, tsq_dtype payload_t,
                    const tsq_params *params, tsq_workspace *ws, void *stream,
                    tsq_stats *stats) {
  if (!ws) return TSQ_ERR_INVALID;
  tsq_status st = check_args(n, key_t, payload_t);
  if (st != TSQ_OK) return st;
  if ((payload_t == TSQ_U32) != (payload != nullptr)) return TSQ_ERR_INVALID;
  if (n > 0 && !keys) return TSQ_ERR_INVALID;
  const int kb = key_bytes_of(key_t);
  if (!element_aligned(keys, kb) || !element_aligned(payload, 4)) return TSQ_ERR_INVALID;
  st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard guard(ws);
  DeviceGuard dg(ws->device);
  if (!dg.ok) return TSQ_ERR_CUDA;
  NvtxRange nvtx("tsq_sort");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n <= 1) {
    if (stats) stats->n = n;
    return TSQ_OK;
  }
  const bool pay = payload_t == TSQ_U32;
  KernelSet ks;
  if (!get_set(key_t, pay, &ks)) return TSQ_ERR_UNSUPPORTED_DTYPE;
  tsq_params defaults;
  memset(&defaults, 0, sizeof(defaults));
  defaults.mitigation = 1;
  defaults.fast_paths = 1;
  const tsq_params &pp = params ? *params : defaults;
  int small_t = default_small_t(key_t, payload_t, n);
#ifdef TSQ_SMALL_T
  small_t = TSQ_SMALL_T;
#endif
  if (pp.small_threshold > 0)
    small_t = pp.small_threshold < ks.small_cap[2] ? pp.small_threshold : ks.small_cap[2];
  // stage export: host-driven levels, the sort in an internal copy, the
  // caller's buffers a view of each level's post-stage state
  const bool exporting = pp.stage_export != 0;
  const bool staged = exporting || !bulk_aligned(keys) || !bulk_aligned(payload);
  const bool host_levels = pp.host_levels || exporting;
  // allocation precedes any mutation (core.py:1599, TempAllocationError)
  st = reserve_locked(ws, n, key_t, payload_t, small_t, staged, exporting);
  if (st != TSQ_OK) return st;
  const Layout L = make_layout(n, key_t, payload_t, small_t, staged, exporting);
  char *base = reinterpret_cast<char *>(ws->block);
  void *skeys = staged ? base + L.stage_keys : keys;
  void *spay = staged && pay ? base + L.stage_pay : payload;
  Params pv;
  fill_params(ws, L, &pv, skeys, spay, n);
  pv.small_t = small_t;
  pv.raw[1] = ks.raw_order ? 1 : 0;
  for (int c = 0; c < kSmallClasses; ++c) pv.sq_lim[c] = ks.small_cap[c];
  pv.dran = pp.dran > 0.0 ? pp.dran : 1.0;
  pv.mitigation = pp.mitigation;
  pv.fast_paths = pp.fast_paths;
  pv.reproducible = pp.reproducible != 0;
  pv.max_depth = pp.max_depth > 0 ? pp.max_depth : default_max_depth(n);
  if (exporting) {
    pv.view_keys = keys;
    pv.view_pay = reinterpret_cast<uint32_t *>(payload);
    pv.stage_out = reinterpret_cast<StageRecord *>(base + L.stage_out);
  }
  TSQ_CUDA(cudaStreamWaitEvent(s, ws->done, 0));
  if (staged) {
    TSQ_CUDA(cudaMemcpyAsync(skeys, keys, n * kb, cudaMemcpyDeviceToDevice, s));
    if (pay) TSQ_CUDA(cudaMemcpyAsync(spay, payload, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  auto stage_back = [&]() -> tsq_status {
    if (staged) {
      TSQ_CUDA(cudaMemcpyAsync(keys, skeys, n * kb, cudaMemcpyDeviceToDevice, s));
      if (pay) TSQ_CUDA(cudaMemcpyAsync(payload, spay, n * 4, cudaMemcpyDeviceToDevice, s));
    }
    return TSQ_OK;
  };

  const int gkey = key_t * 2 + (pay ? 1 : 0);
  if (!host_levels) {
    GraphEntry &ge = ws->graphs[gkey];
    if (!ge.exec) {
      st = build_graph(ws, key_t, pay, &ge);
      if (st != TSQ_OK) {
        ws->graphs.erase(gkey);
        return st;
      }
    }
    pv.use_cond = 1;
    pv.cond = ge.cond;
    pv.cond_outer = ge.cond_outer;
    Params *dst = ws->d_params;
    void *args[2] = {&pv, &dst};
    cudaKernelNodeParams kp = ge.init_params;
    kp.kernelParams = args;
    TSQ_CUDA(cudaGraphExecKernelNodeSetParams(ge.exec, ge.init_node, &kp));
    TSQ_CUDA(cudaGraphLaunch(ge.exec, s));
    st = stage_back();
    if (st != TSQ_OK) return st;
    TSQ_CUDA(cudaEventRecord(ws->done, s));
    if (stats) {
      st = read_ctl(ws, s);
      if (st != TSQ_OK) return st;
      st = fill_stats(ws, n, stats);
      cudaEventElapsedTime(&stats->ms_levels, ge.ev[1], ge.ev[2]);
      cudaEventElapsedTime(&stats->ms_total, ge.ev[0], ge.ev[2]);
      return st;
    }
    return TSQ_OK;
  }

  // host-driven levels: same kernels, one launch per level with a read-back
  // of the queue size in between (per-level timing / trace / stage export)
  st = prepare_small_smem(ks);
  if (st != TSQ_OK) return st;
  TSQ_CUDA(cudaFuncSetAttribute(ks.exportk, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
  pv.use_cond = 0;
  struct Events {
    cudaEvent_t e[5] = {};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev;
  for (auto &x : ev.e) TSQ_CUDA(cudaEventCreate(&x));
  cudaEvent_t &e0 = ev.e[0], &em = ev.e[1], &e1 = ev.e[2], &t0 = ev.e[3], &t1 = ev.e[4];
  ws->level_ms.clear();
  ws->sched_ms.clear();
  ws->level_segs.clear();
  ws->level_tiles.clear();
  Params *dst = ws->d_params;
  TSQ_CUDA(cudaEventRecord(t0, s));
  void *iargs[2] = {&pv, &dst};
  TSQ_CUDA(cudaLaunchKernel(ks.init, dim3(1), dim3(kThreads), iargs, 0, s));
  void *largs[2] = {&dst, &ws->d_ctl};
  const LevelLaunch LL = level_launch(ws, ks);
  float total_levels = 0.f;
  ws->level_bytes.clear();
  u64 bytes_before = 0;
  for (int lv = 0; lv < kMaxLevels; ++lv) {
    st = read_ctl(ws, s);
    if (st != TSQ_OK) return st;
    if (lv > 0) {  // algorithmic bytes the previous level's partition pass moved
      ws->level_bytes.push_back(ws->h_ctl->bytes_partition - bytes_before);
      bytes_before = ws->h_ctl->bytes_partition;
    }
    if (ws->h_ctl->flush) {  // the queues are near full: drain them, then go on
      TSQ_CUDA(launch_drain(ws, ks, &dst, s));
      st = read_ctl(ws, s);
      if (st != TSQ_OK) return st;
    }
    if (getenv("TSQ_DEBUG_LEVELS"))
      fprintf(stderr, "tsq level %d: segments %u tiles %u small %u/%u runs %u error %u\n", lv,
              ws->h_ctl->cur_nseg, ws->h_ctl->cur_ntiles, ws->h_ctl->sq_count[0],
              ws->h_ctl->sq_count[1], (uint32_t)(ws->h_ctl->run_packed >> 32), ws->h_ctl->error);
    if (ws->h_ctl->cur_nseg == 0 || ws->h_ctl->error) break;
    const uint32_t nseg = ws->h_ctl->cur_nseg;
    ws->level_segs.push_back(nseg);
    ws->level_tiles.push_back(ws->h_ctl->cur_ntiles);
    char name[32];
    snprintf(name, sizeof(name), "tsq level %d", lv);
    NvtxRange lvl(name);
    TSQ_CUDA(cudaEventRecord(e0, s));
    TSQ_CUDA(cudaLaunchKernel(ks.part, LL.part_grid, dim3(kPartThreads), largs, ks.part_smem, s));
    TSQ_CUDA(cudaEventRecord(em, s));
    if (exporting) {
      const unsigned g = nseg < 4u * (unsigned)ws->num_sms ? nseg : 4u * (unsigned)ws->num_sms;
      TSQ_CUDA(cudaLaunchKernel(ks.exportk, dim3(g), dim3(kThreads), largs, 0, s));
    }
    TSQ_CUDA(cudaLaunchKernel(ks.sched, LL.sched_grid, dim3(kThreads), largs, ks.sched_smem, s));
    TSQ_CUDA(cudaEventRecord(e1, s));
    TSQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f, ms2 = 0.f;
    cudaEventElapsedTime(&ms, e0, em);
    cudaEventElapsedTime(&ms2, em, e1);
    ws->level_ms.push_back(ms);
    ws->sched_ms.push_back(ms2);
    total_levels += ms + ms2;
    if (exporting) {
      ws->records.resize(nseg);
      TSQ_CUDA(cudaMemcpyAsync(ws->records.data(), pv.stage_out, nseg * sizeof(StageRecord),
                               cudaMemcpyDeviceToHost, s));
      TSQ_CUDA(cudaStreamSynchronize(s));
      if (pp.on_level) pp.on_level(pp.on_level_user, lv, ws->records.data(), nseg);
    }
  }
  TSQ_CUDA(launch_drain(ws, ks, &dst, s));
  st = stage_back();
  if (st != TSQ_OK) return st;
  TSQ_CUDA(cudaEventRecord(t1, s));
  TSQ_CUDA(cudaEventRecord(ws->done, s));
  st = read_ctl(ws, s);
  if (st == TSQ_OK && stats) {
    st = fill_stats(ws, n, stats);
    stats->ms_levels = total_levels;
    cudaEventElapsedTime(&stats->ms_total, t0, t1);
  } else if (st == TSQ_OK) {
    st = status_of(ws->h_ctl->error);
  }
  return st;
}

int tsq_level_trace(const tsq_workspace *ws, float *part_ms, float *sched_ms, uint32_t *segs,
                    uint32_t *tiles, uint64_t *bytes, int cap) {
  if (!ws) return 0;
  int n = (int)ws->level_ms.size();
  for (int i = 0; i < n && i < cap; ++i) {
    if (bytes) bytes[i] = i < (int)ws->level_bytes.size() ? ws->level_bytes[i] : 0;
    if (part_ms) part_ms[i] = ws->level_ms[i];
    if (sched_ms) sched_ms[i] = ws->sched_ms[i];
    if (segs) segs[i] = ws->level_segs[i];
    if (tiles) tiles[i] = ws->level_tiles[i];
  }
  return n;
}

tsq_status tsq_partition_segment(const void *keys, const void *payload, void *out_keys,
                                 void *out_payload, size_t n, tsq_dtype key_t,
                                 tsq_dtype payload_t, uint64_t pivot, tsq_workspace *ws,
                                 void *stream, int64_t *new_l, int64_t *new_r) {
  if (!ws || !new_l || !new_r) return TSQ_ERR_INVALID;
  tsq_status st = check_args(n, key_t, payload_t);
  if (st != TSQ_OK) return st;
  const bool pay = payload_t == TSQ_U32;
  if (pay != (payload != nullptr) || pay != (out_payload != nullptr)) return TSQ_ERR_INVALID;
  const int kb = key_bytes_of(key_t);
  if (!element_aligned(keys, kb) || !element_aligned(out_keys, kb) ||
      !element_aligned(payload, 4) || !element_aligned(out_payload, 4))
    return TSQ_ERR_INVALID;
  if (n == 0) {
    *new_l = -1;
    *new_r = 0;
    return TSQ_OK;
  }
  st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard guard(ws);
  DeviceGuard dg(ws->device);
  if (!dg.ok) return TSQ_ERR_CUDA;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // a misaligned output is written through an aligned copy (bulk stores)
  const bool staged = !bulk_aligned(out_keys) || !bulk_aligned(out_payload);
  st = reserve_locked(ws, n, key_t, payload_t, 0, staged);
  if (st != TSQ_OK) return st;
  KernelSet ks;
  if (!get_set(key_t, pay, &ks)) return TSQ_ERR_UNSUPPORTED_DTYPE;
  const Layout L = make_layout(n, key_t, payload_t, 0, staged);
  char *base = reinterpret_cast<char *>(ws->block);
  void *ok = staged ? base + L.stage_keys : out_keys;
  void *op = staged && pay ? base + L.stage_pay : out_payload;
  Params pv;
  fill_params(ws, L, &pv, ok, op, n);
  pv.keys[1] = const_cast<void *>(keys);
  pv.pay[1] = reinterpret_cast<uint32_t *>(const_cast<void *>(payload));
  pv.raw[1] = 1;
  pv.aligned[1] = bulk_aligned(keys) && bulk_aligned(payload);
  pv.single_stage = 1;
  pv.given_pivot = host_enc(key_t, pivot);
  pv.use_cond = 0;
  TSQ_CUDA(cudaStreamWaitEvent(s, ws->done, 0));
  Params *dst = ws->d_params;
  void *iargs[2] = {&pv, &dst};
  TSQ_CUDA(cudaLaunchKernel(ks.init, dim3(1), dim3(kThreads), iargs, 0, s));
  void *largs[2] = {&dst, &ws->d_ctl};
  st = prepare_small_smem(ks);
  if (st != TSQ_OK) return st;
  TSQ_CUDA(launch_level(ks, level_launch(ws, ks), &dst, &ws->d_ctl, s));
  TSQ_CUDA(cudaLaunchKernel(ks.retire, dim3(occupancy_grid(ws, ks.retire, 0)), dim3(kThreads),
                            largs, 0, s));
  if (staged) {
    TSQ_CUDA(cudaMemcpyAsync(out_keys, ok, n * kb, cudaMemcpyDeviceToDevice, s));
    if (pay) TSQ_CUDA(cudaMemcpyAsync(out_payload, op, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  TSQ_CUDA(cudaEventRecord(ws->done, s));
  st = read_ctl(ws, s);
  if (st != TSQ_OK) return st;
  if (ws->h_ctl->error) return TSQ_ERR_CAPACITY;
  *new_l = (int64_t)ws->h_ctl->stage_lt - 1;
  *new_r = (int64_t)n - (int64_t)ws->h_ctl->stage_gt;
  return TSQ_OK;
}

tsq_status tsq_select_pivot(const void *keys, size_t n, tsq_dtype key_t, double dran,
                            int32_t mitigation, tsq_workspace *ws, void *stream,
                            uint64_t *pivot, int32_t *order_flag) {
  if (!ws || !pivot || !order_flag) return TSQ_ERR_INVALID;
  tsq_status st = check_args(n, key_t, TSQ_NONE);
  if (st != TSQ_OK) return st;
  if (n < 2) return TSQ_ERR_INVALID;
  if (!element_aligned(keys, key_bytes_of(key_t))) return TSQ_ERR_INVALID;
  st = acquire(ws);
  if (st != TSQ_OK) return st;
  ActiveGuard guard(ws);
  DeviceGuard dg(ws->device);
  if (!dg.ok) return TSQ_ERR_CUDA;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  KernelSet ks;
  if (!get_set(key_t, false, &ks)) return TSQ_ERR_UNSUPPORTED_DTYPE;
  Params pv;
  memset(&pv, 0, sizeof(pv));
  pv.keys[0] = const_cast<void *>(keys);
  pv.raw[0] = 1;
  pv.n = (long long)n;
  pv.dran = dran > 0.0 ? dran : 1.0;
  pv.mitigation = mitigation;
  pv.ctl = ws->d_ctl;
  TSQ_CUDA(cudaStreamWaitEvent(s, ws->done, 0));
  void *args[1] = {&pv};
  TSQ_CUDA(cudaLaunchKernel(ks.selp, dim3(1), dim3(kThreads), args, 0, s));
  TSQ_CUDA(cudaEventRecord(ws->done, s));
  st = read_ctl(ws, s);
  if (st != TSQ_OK) return st;
  const int kb = key_bytes_of(key_t);
  *pivot = kb == 4 ? (ws->h_ctl->stage_lt & 0xffffffffull) : ws->h_ctl->stage_lt;
  *order_flag = (int32_t)(long long)ws->h_ctl->stage_gt;
  return TSQ_OK;
}

tsq_status tsq_apply_permutation(const void *src_rows, void *dst_rows, size_t n,
                                 size_t row_bytes, const uint32_t *perm, void *stream) {
  if (n == 0 || row_bytes == 0) return TSQ_OK;
  if (!src_rows || !dst_rows || !perm || src_rows == dst_rows) return TSQ_ERR_INVALID;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uintptr_t a = (uintptr_t)src_rows | (uintptr_t)dst_rows | (uintptr_t)row_bytes;
  int mode = (a % 16 == 0) ? 2 : ((a % 4 == 0) ? 1 : 0);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t want = (n + 7) / 8;  // 8 warps (rows in flight) per CTA
  const unsigned grid = (unsigned)(want < (size_t)sms * 8 ? want : (size_t)sms * 8);
  gather_rows_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const unsigned char *>(src_rows),
                                          reinterpret_cast<unsigned char *>(dst_rows), perm, n,
                                          row_bytes, mode);
  TSQ_CUDA(cudaGetLastError());
  return TSQ_OK;
}

}  // extern "C"

#ifdef TSQ_TRACE
// Profiling builds only (libtsq_b200_trace.so): per-tile timeline of one
// level of the partition pass, read back by scripts/trace_level.py.
extern "C" int tsq_trace_set_level(int level) {
  return cudaMemcpyToSymbol(tsq::g_trace_level, &level, sizeof(int)) == cudaSuccess ? 0 : -1;
}
extern "C" int tsq_trace_copy(void *dst, size_t bytes) {
  const size_t cap = sizeof(tsq::g_trace);
  if (bytes > cap) bytes = cap;
  if (cudaMemset(nullptr, 0, 0) != cudaSuccess) cudaGetLastError();
  return cudaMemcpyFromSymbol(dst, tsq::g_trace, bytes) == cudaSuccess ? 0 : -1;
}
extern "C" int tsq_trace_clear(void) {
  void *p = nullptr;
  if (cudaGetSymbolAddress(&p, tsq::g_trace) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(tsq::g_trace)) == cudaSuccess ? 0 : -1;
}
#endif
