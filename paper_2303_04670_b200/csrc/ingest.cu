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
    const int c = p[e] > 0 ? 0 : 1;  // channel 0: p > 0, channel 1: the rest (events.py:267-272)
    atomicAdd(vals + ((int64_t)c * H + y[e]) * W + x[e], i < na ? -1.0f : 1.0f);
  }
}

// ---- batched per-step ingest of S sessions into device rings (serving.EventPipeline) ----------
// desc[s] = {first record of session s in the step's record block, new records, absolute index of
// its first new event}; the session's ring holds events at slot (absolute index) & (R - 1).
__global__ void __launch_bounds__(256) k_ingest_ring(const uint8_t* __restrict__ rec, const int64_t* __restrict__ desc,
                                                     int64_t R, uint64_t* t, uint16_t* x, uint16_t* y, int8_t* p) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  const int64_t first = desc[3 * s], n = desc[3 * s + 1], head = desc[3 * s + 2];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = rec + (first + e) * 13;
    uint64_t tv = 0;
#pragma unroll
    for (int k = 7; k >= 0; --k) tv = (tv << 8) | r[k];
    const int64_t slot = (int64_t)s * R + ((head + e) & (R - 1));
    t[slot] = tv;
    x[slot] = (uint16_t)(r[8] | (r[9] << 8));
    y[slot] = (uint16_t)(r[10] | (r[11] << 8));
    p[slot] = (int8_t)r[12];
  }
}

// count (2 ch) and / or timestamp (2 ch) encodings of every session's window [lo, hi) (absolute
// event indices) into out[s] (zeroed by the caller).  Both are order-free: integer counts in f32
// (+1 adds are exact below 2^24) and a max of non-negative floats (int compare of the bits), so the
// scatter is bit-identical to np.add.at / np.maximum.at (events.py:267-280).
__global__ void __launch_bounds__(256) k_encode_windows(const uint64_t* __restrict__ t, const uint16_t* __restrict__ x,
                                                        const uint16_t* __restrict__ y, const int8_t* __restrict__ p,
                                                        int64_t R, const int64_t* __restrict__ win, int H, int W,
                                                        int mode, float* out, int64_t os) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  const int64_t lo = win[4 * s], hi = win[4 * s + 1], t0 = win[4 * s + 2] - win[4 * s + 3];
  const double dd = (double)win[4 * s + 3];
  const int64_t HW = (int64_t)H * W;
  float* o = out + (int64_t)s * os;
  float* ts = o + ((mode & 1) ? 2 * HW : 0);
  for (int64_t e = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < hi; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t slot = (int64_t)s * R + (e & (R - 1));
    const int64_t px = (p[slot] > 0 ? 0 : HW) + (int64_t)y[slot] * W + x[slot];
    if (mode & 1) atomicAdd(o + px, 1.0f);
    if (mode & 2) {
      const float rel = (float)(((double)t[slot] - (double)t0) / dd);  // f32((t - (tau - delta)) / delta in f64)
      atomicMax(reinterpret_cast<int*>(ts + px), __float_as_int(rel));
    }
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

int evc_ingest_ring(const uint8_t* records, const int64_t* desc, int64_t max_new, int64_t ring, uint64_t* t,
                    uint16_t* x, uint16_t* y, int8_t* p, int32_t S, void* stream) {
  EVC_CHECK_ARG(desc && t && x && y && p && S > 0 && ring > 0 && (ring & (ring - 1)) == 0 && max_new >= 0,
                "ingest_ring: bad argument (ring must be a power of two)");
  EVC_CHECK_ARG(max_new <= ring, "ingest_ring: more new events than the ring holds");
  if (max_new == 0) return EVC_OK;
  EVC_CHECK_ARG(records != nullptr, "ingest_ring: null records");
  const int gx = (int)std::min<int64_t>((max_new + 255) / 256, 64);
  launch_pdl(k_ingest_ring, dim3(gx, S), dim3(256), 0, as_stream(stream), records, desc, ring, t, x, y, p);
  EVC_LAUNCH_CHECK("ingest_ring");
  return EVC_OK;
}

int evc_encode_windows(const uint64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t ring,
                       const int64_t* win, int64_t max_events, int32_t H, int32_t W, int32_t mode, float* out,
                       int64_t out_stride, int32_t S, void* stream) {
  EVC_CHECK_ARG(t && x && y && p && win && out && S > 0 && H > 0 && W > 0 && ring > 0 && (ring & (ring - 1)) == 0,
                "encode_windows: bad argument");
  EVC_CHECK_ARG(mode >= 1 && mode <= 3, "encode_windows: mode = 1 (count), 2 (timestamp) or 3 (count + timestamp)");
  const int64_t C = mode == 3 ? 4 : 2;
  EVC_CHECK_ARG(out_stride >= C * H * W && max_events <= ring, "encode_windows: output stride / window size");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemset2DAsync(out, (size_t)out_stride * 4, 0, (size_t)C * H * W * 4, (size_t)S, st);
  if (e != cudaSuccess) {
    set_error(std::string("evc: encode_windows memset: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  if (max_events <= 0) return EVC_OK;
  const int gx = (int)std::min<int64_t>((max_events + 255) / 256, 128);
  launch_pdl(k_encode_windows, dim3(gx, S), dim3(256), 0, st, t, x, y, p, ring, win, (int)H, (int)W, (int)mode, out,
             out_stride);
  EVC_LAUNCH_CHECK("encode_windows");
  return EVC_OK;
}

}  // extern "C"
