// Shared helpers for libevconv (sm_100a).  Internal header.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/evconv.h"

namespace evc {

void set_error(const std::string& msg);

#define EVC_CHECK_ARG(cond, msg)                 \
  do {                                           \
    if (!(cond)) {                               \
      ::evc::set_error(std::string("evc: ") + (msg)); \
      return EVC_EINVAL;                         \
    }                                            \
  } while (0)

#define EVC_LAUNCH_CHECK(what)                                              \
  do {                                                                      \
    cudaError_t e__ = cudaGetLastError();                                   \
    if (e__ != cudaSuccess) {                                               \
      ::evc::set_error(std::string("evc: ") + (what) + ": " + cudaGetErrorString(e__)); \
      return EVC_ECUDA;                                                     \
    }                                                                       \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (evc_set_pdl): step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs may start
// while its predecessor drains.  EVERY kernel launched that way executes pdl_wait()
// before touching data an earlier kernel writes (which also keeps the dependency
// transitive down the stream); pdl_trigger() lets the successor launch early.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// cudaLaunchKernelEx with the PDL attribute when enabled.
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

static inline int cdiv(int a, int b) { return (a + b - 1) / b; }
static inline int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Geometry of a tile grid.
struct Grid {
  int C, H, W, th, tw, GH, GW;
};

static inline Grid grid_of(const evc_tensor& t) {
  Grid g;
  g.C = t.C;
  g.H = t.H;
  g.W = t.W;
  g.th = t.th;
  g.tw = t.tw;
  g.GH = (t.H + t.th - 1) / t.th;
  g.GW = (t.W + t.tw - 1) / t.tw;
  return g;
}

// Device view of an evc_tensor (passed by value to kernels).
struct TView {
  float* v;
  uint8_t* f;
  int64_t vs, fs;
  int C, H, W, th, tw, GH, GW;
  __host__ __device__ __forceinline__ float* plane(int s, int c) const {
    return v + (int64_t)s * vs + (int64_t)c * H * W;
  }
  __host__ __device__ __forceinline__ uint8_t* fplane(int s, int c) const {
    return f + (int64_t)s * fs + (int64_t)c * GH * GW;
  }
};

static inline TView view_of(const evc_tensor& t) {
  TView r;
  r.v = t.vals;
  r.f = t.flags;
  r.vs = t.vstride;
  r.fs = t.fstride;
  r.C = t.C;
  r.H = t.H;
  r.W = t.W;
  r.th = t.th;
  r.tw = t.tw;
  r.GH = (t.H + t.th - 1) / t.th;
  r.GW = (t.W + t.tw - 1) / t.tw;
  return r;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024).  Result valid in thread 0.
template <typename T, typename F>
__device__ __forceinline__ T block_sum(T v, F wsum) {
  __shared__ T red[32];
  v = wsum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    r = lane < nw ? red[lane] : T(0);
    r = wsum(r);
  }
  return r;
}

// Channels-innermost hi/lo shadow of a conv input (the TMA A operand of
// conv_fused.cu): pixel p owns 2*cp floats, the TF32 head of channel c at
// [p*2cp + c] and the tail x - head at [p*2cp + cp + c]; cp = channels padded to
// a multiple of 32 so both 32-channel boxes start 128-byte aligned.
// 4-byte global -> shared copy that does not wait for the load (LDGSTS); completed by
// cp_async_wait_all() before the barrier that publishes the staged data.
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// floor(a / d) for 0 <= a < 2^22 through an fp32 reciprocal: (a + 0.5) is exact and the
// relative error of (a + 0.5) * RN(1/d) is <= 2^-23, i.e. below a * 2^-23 / d < 0.5 / d, the
// distance of (a + 0.5) / d to the next integer -- so the truncation is exact.
// Replaces the ~20-instruction integer division in per-element index math.
struct FDiv {
  float inv;
  int d;
};
__device__ __forceinline__ FDiv fdiv_of(int d) { return FDiv{__frcp_rn((float)d), d}; }
__device__ __forceinline__ int fdiv(int a, const FDiv& f) { return __float2int_rz(__fmul_rn((float)a + 0.5f, f.inv)); }

__device__ __forceinline__ float tf32_head(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// Shadow pixel layout: with cp a multiple of 32 (the TMA path), 32-channel chunks of
// [32 heads | 32 tails] -- a channel's tail sits 128 bytes after its head (one base register,
// immediate offsets) and a TMA box of heads (or tails) is 32 consecutive floats; otherwise
// (the CUDA-core path's cp = 4-aligned C) one chunk [cp heads | cp tails].
// cp < 0 selects an fp32 shadow of -cp channels, [values] per pixel: the CUDA-core thin
// conv reads the value itself (head + tail rebuilt it exactly), so it needs half the bytes.
__host__ __device__ __forceinline__ int hwc_px(int cp) { return cp < 0 ? -cp : 2 * cp; }
__device__ __forceinline__ int hwc_head(int cp, int c) {
  return cp > 0 && (cp & 31) == 0 ? ((c >> 5) << 6) + (c & 31) : c;
}
// Offset of a channel's tail from its head.  Only defined for the hi/lo layouts (cp > 0): an fp32
// shadow (cp < 0) has no tails, and a negative offset would address the previous pixel -- trap.
__device__ __forceinline__ int hwc_unit(int cp) {
  if (cp <= 0) __trap();
  return (cp & 31) == 0 ? 32 : cp;
}
__device__ __forceinline__ void hwc_store(float* pix, int cp, int c, float x) {
  if (cp < 0) {
    pix[c] = x;
    return;
  }
  const float h = tf32_head(x);
  const int o = hwc_head(cp, c);
  pix[o] = h;
  pix[o + hwc_unit(cp)] = __fsub_rn(x, h);
}

// Activation f of inc_activation (tensors.py:285-312), float32 ops with the
// reference's rounding (no FMA contraction).
__device__ __forceinline__ float act_apply(float x, int kind, float alpha) {
  switch (kind) {
    case EVC_ACT_RELU:
      return fmaxf(x, 0.0f);
    case EVC_ACT_SIGMOID:
      return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
    case EVC_ACT_TANH:
      return tanhf(x);
    default:
      return x > 0.0f ? x : __fmul_rn(alpha, x);
  }
}

// Bilinear upsampling taps of one output coordinate: half-pixel source
// (i + 0.5) / f - 0.5, clamped, float32 weights (tensors.py:259-266).
struct Tap {
  int i0, i1;
  float w0, w1;
};

__device__ __forceinline__ Tap bilinear_tap(int o, int n_in, int f) {
  const float src = __fsub_rn(__fdiv_rn(__fadd_rn((float)o, 0.5f), (float)f), 0.5f);
  const float fl = floorf(src);
  const float frac = __fsub_rn(src, fl);
  Tap t;
  const int i0 = (int)fl;
  t.i1 = min(max(i0 + 1, 0), n_in - 1);
  t.i0 = min(max(i0, 0), n_in - 1);
  t.w1 = frac;
  t.w0 = __fsub_rn(1.0f, frac);
  return t;
}

// Upsampled value of output (u, v) from plane xv (H x W input), float32 op
// order of dense_upsample (tensors.py:269-282): rows first, then columns.
__device__ __forceinline__ float upsample_at(const float* xv, int H, int W, int u, int v, int f, int mode) {
  if (mode == 0) return xv[(int64_t)(u / f) * W + v / f];
  const Tap tr = bilinear_tap(u, H, f), tc = bilinear_tap(v, W, f);
  const float* x0 = xv + (int64_t)tr.i0 * W;
  const float* x1 = xv + (int64_t)tr.i1 * W;
  const float ra = __fadd_rn(__fmul_rn(x0[tc.i0], tr.w0), __fmul_rn(x1[tc.i0], tr.w1));
  const float rb = __fadd_rn(__fmul_rn(x0[tc.i1], tr.w0), __fmul_rn(x1[tc.i1], tr.w1));
  return __fadd_rn(__fmul_rn(ra, tc.w0), __fmul_rn(rb, tc.w1));
}

// Input tile box [lo, hi] (in tile units) read by the upsampled output range [o0, o1).
__device__ __forceinline__ void upsample_box(int o0, int o1, int n_in, int f, int mode, int tile, int& lo,
                                             int& hi) {
  if (mode == 0) {
    lo = (o0 / f) / tile;
    hi = ((o1 - 1) / f) / tile;
  } else {
    lo = bilinear_tap(o0, n_in, f).i0 / tile;
    hi = bilinear_tap(o1 - 1, n_in, f).i1 / tile;
  }
}

// Sum each session's partials in a fixed order, then the EMA / k update
// (sparsify.py:72-76) or the reset (sparsify.py:43-51).  One CTA does all S.
__device__ __forceinline__ void sparsify_finalize_all(const double* partials, int64_t n, double* norm_ema, double* kdev, double tp,
                                      double decay, int reset, int S, int s_first = 0) {
  for (int s = s_first; s < S; ++s) {
    double sum = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) sum += ((volatile const double*)partials)[(int64_t)s * n + e];
    sum = block_sum<double>(sum, [](double v) { return warp_sum_d(v); });
    if (threadIdx.x == 0) {
      // np.linalg.norm of float32 data returns float32 (sparsify.py:49,73)
      const double norm = (double)__double2float_rn(sqrt(sum));
      const double ne =
          reset ? norm : __dadd_rn(__dmul_rn(decay, norm_ema[s]), __dmul_rn(__dsub_rn(1.0, decay), norm));
      norm_ema[s] = ne;
      if (tp > 0.0) kdev[s] = __dmul_rn(tp, ne);
    }
    __syncthreads();
  }
}

}  // namespace evc

namespace evc {
// Per-translation-unit module loaders (force lazy-loaded modules in before
// any CUDA-graph capture).
int init_masks();
int init_conv();
int init_conv_mask();
int init_conv_fused();
int init_conv_scatter();
int init_subpixel();
int init_elementwise();
int init_bands();
int init_upsparsify();
int init_linear_events();
}  // namespace evc
