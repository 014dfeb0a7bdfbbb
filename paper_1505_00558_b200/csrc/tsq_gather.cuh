// tsq_gather.cuh -- late swapping for large elements (the reference's
// bigelem.py: sort position handles first, then move every element once;
// /root/reference/pkg/src/tsqsort/bigelem.py:31-99, dispatched from
// core.py:1595-1598 when element_size >= late_swap_byte_threshold).
//
// On the device the handle sort is the ordinary (key, uint32 index) records
// sort; the permutation is then applied as one coalesced gather instead of
// _apply's cycle walk: dst[i] = src[perm[i]] for rows of `row_bytes`.  One
// warp moves one row per step with 16-byte vectors when rows and both bases
// are 16-byte aligned (else 4-byte words, else bytes).  HBM-bound: n *
// row_bytes read + written.
#pragma once

namespace tsq {

template <typename W>
__device__ __forceinline__ void copy_row(const unsigned char *src, unsigned char *dst,
                                         size_t bytes, int lane) {
  const W *s = reinterpret_cast<const W *>(src);
  W *d = reinterpret_cast<W *>(dst);
  const size_t nw = bytes / sizeof(W);
  for (size_t w = (size_t)lane; w < nw; w += 32) d[w] = __ldg(s + w);
}

// dst row i <- src row perm[i]; mode 2: uint4 words, 1: uint32, 0: bytes
__global__ void __launch_bounds__(256) gather_rows_kernel(const unsigned char *__restrict__ src,
                                                          unsigned char *__restrict__ dst,
                                                          const uint32_t *__restrict__ perm,
                                                          size_t n, size_t row_bytes, int mode) {
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t r = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const size_t from = (size_t)__ldg(perm + r);
    const unsigned char *s = src + from * row_bytes;
    unsigned char *d = dst + r * row_bytes;
    if (mode == 2) copy_row<uint4>(s, d, row_bytes, lane);
    else if (mode == 1) copy_row<uint32_t>(s, d, row_bytes, lane);
    else copy_row<unsigned char>(s, d, row_bytes, lane);
  }
}

}  // namespace tsq
