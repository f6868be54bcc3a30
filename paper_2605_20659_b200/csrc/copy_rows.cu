// Segmented row copy: the pack / unpack of the sequence <-> head all-to-alls
// around the op (ulysses.py, BASELINE config 4) as one launch each.
//
// A segment copies `rows` rows of `row_bytes` bytes from src (rows
// src_stride bytes apart) to dst (dst_stride apart); segment k covers the
// global rows [row0_k, row0_k + rows_k) of the launch, row0 ascending.  One
// warp per row, 16-byte vectors: a head's [L, d] slice of a [B, L, H, d]
// tensor is a segment of 256-byte rows H * d * 2 bytes apart.
#include <cuda_runtime.h>

#include "common.cuh"

namespace ropeslr {

__global__ void __launch_bounds__(256) copy_rows_kernel(const ropeslr_row_segment* __restrict__ segs, int nseg,
                                                        int64_t total) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < total;
       row += warps) {
    int lo = 0, hi = nseg - 1;  // last segment with row0 <= row
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].row0 <= row) lo = mid;
      else hi = mid - 1;
    }
    const ropeslr_row_segment sg = segs[lo];
    const int64_t r = row - sg.row0;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const char*>(sg.src) + r * sg.src_stride);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(sg.dst) + r * sg.dst_stride);
    for (int c = lane; c < sg.row_bytes / 16; c += 32) dst[c] = src[c];
  }
}

}  // namespace ropeslr

extern "C" int ropeslr_copy_rows(const ropeslr_row_segment* segs, int32_t nseg, int64_t total_rows, void* stream) {
  if (nseg < 0 || total_rows < 0) return ROPESLR_ERR_SHAPE;
  if (nseg == 0 || total_rows == 0) return ROPESLR_OK;
  if (segs == nullptr) return ROPESLR_ERR_NULL;
  const int64_t blocks = ropeslr::ceil_div(total_rows, 8);
  const int64_t cap = 16 * static_cast<int64_t>(ropeslr::num_sms());
  ropeslr::copy_rows_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0,
                              static_cast<cudaStream_t>(stream)>>>(segs, nseg, total_rows);
  return ropeslr::launch_status();
}
