// Event ingest on the device.
//
// * evc_unpack_events: the EVB record stream (events.py:35-37: little-endian
//   {u64 t, u16 x, u16 y, i8 p}, 13 bytes, no padding) is uploaded as raw bytes and
//   split into the t / x / y / p columns the binning kernel reads, so the host never
//   touches individual events (read_events' numpy record view, events.py:185-206,
//   is the reference).
// * evc_count_increment: the increment of the `count` encoding between two windows
//   of one stream, from only the events that leave and enter:
//     encode(cur) - encode(prev) = +1 per entering event - 1 per leaving event
//   on channel 0 (p > 0) or 1 (p < 0) (events.py:267-272).  Counts are integers in
//   float32, so the scatter of +-1 is exact and order-free, and the result equals
//   step_increment(encode(prev), encode(cur)) bit for bit (an add of +1 and -1 gives
//   +0, the value of cur - prev for unchanged counts).  The tile mask is then made
//   from the values (make_tile_mask).

#include <algorithm>

#include "common.cuh"

namespace evc {

__global__ void __launch_bounds__(256) k_unpack_events(const uint8_t* __restrict__ rec, int64_t n, uint64_t* t,
                                                       uint16_t* x, uint16_t* y, int8_t* p) {
  pdl_wait();
  pdl_trigger();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = rec + e * 13;
    uint64_t tv = 0;
#pragma unroll
    for (int k = 7; k >= 0; --k) tv = (tv << 8) | r[k];
    t[e] = tv;
    x[e] = (uint16_t)(r[8] | (r[9] << 8));
    y[e] = (uint16_t)(r[10] | (r[11] << 8));
    p[e] = (int8_t)r[12];
  }
}

// events [a0, a1) add -1, [b0, b1) add +1 at (channel of p, y, x) of the (2, H, W) plane
__global__ void __launch_bounds__(256) k_count_scatter(const uint16_t* __restrict__ x, const uint16_t* __restrict__ y,
                                                       const int8_t* __restrict__ p, int64_t a0, int64_t a1,
                                                       int64_t b0, int64_t b1, int H, int W, float* vals) {
  pdl_wait();
  pdl_trigger();
  const int64_t na = a1 - a0, n = na + (b1 - b0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i < na ? a0 + i : b0 + (i - na);
    const int pol = p[e];
    if (pol == 0) continue;  // neither count channel (events.py:269-272)
    const int c = pol > 0 ? 0 : 1;
    atomicAdd(vals + ((int64_t)c * H + y[e]) * W + x[e], i < na ? -1.0f : 1.0f);
  }
}

}  // namespace evc

using namespace evc;

extern "C" {

int evc_unpack_events(const uint8_t* records, int64_t n, uint64_t* t, uint16_t* x, uint16_t* y, int8_t* p,
                      void* stream) {
  EVC_CHECK_ARG(n >= 0 && (n == 0 || (records && t && x && y && p)), "unpack_events: null argument");
  if (n == 0) return EVC_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  launch_pdl(k_unpack_events, dim3(grid), dim3(256), 0, as_stream(stream), records, n, t, x, y, p);
  EVC_LAUNCH_CHECK("unpack_events");
  return EVC_OK;
}

int evc_count_increment(const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t lo_prev, int64_t hi_prev,
                        int64_t lo_cur, int64_t hi_cur, const evc_tensor* out, void* stream) {
  EVC_CHECK_ARG(x && y && p && out && out->vals && out->flags && out->C == 2, "count_increment: bad argument");
  EVC_CHECK_ARG(0 <= lo_prev && lo_prev <= hi_prev && 0 <= lo_cur && lo_cur <= hi_cur && lo_prev <= lo_cur &&
                    hi_prev <= hi_cur,
                "count_increment: windows must move forward in time");
  cudaStream_t st = as_stream(stream);
  // leaving: in prev, not in cur; entering: in cur, not in prev
  const int64_t a0 = lo_prev, a1 = std::min(lo_cur, hi_prev);
  const int64_t b0 = std::max(hi_prev, lo_cur), b1 = hi_cur;
  const int64_t n = (a1 - a0) + (b1 - b0);
  cudaError_t e = cudaMemsetAsync(out->vals, 0, sizeof(float) * 2 * (size_t)out->H * out->W, st);
  if (e != cudaSuccess) {
    set_error(std::string("evc: count_increment memset: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  if (n > 0) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    launch_pdl(k_count_scatter, dim3(grid), dim3(256), 0, st, x, y, p, a0, a1, b0, b1, (int)out->H, (int)out->W,
               out->vals);
    EVC_LAUNCH_CHECK("count_increment");
  }
  return evc_make_tile_mask(out, 1, stream);
}

}  // extern "C"
