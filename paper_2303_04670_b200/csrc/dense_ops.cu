// Dense (unmasked) operators of the dense pass, norm finalize, upsample and
// maxpool (tensors.py:242-312, increment_ops.py:271-310, sparsify.py:43-51).
//
// upsample / maxpool are "band" kernels (one CTA per session x channel x
// output tile-row); masked calls process an output tile when it is live or was
// live last step, so recomputation from zero inputs restores exact zeros.
// Float arithmetic uses _rn intrinsics so no FMA contraction changes the
// reference's float32 rounding sequence.

#include "common.cuh"

namespace evc {

__device__ __forceinline__ float act_f(float x, int kind, float alpha) {
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

__global__ void k_act_dense(const float* __restrict__ x, int64_t xs, float* __restrict__ y, int64_t ys,
                            float* __restrict__ acc, int64_t as, int64_t n, int kind, float alpha) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[(int64_t)s * xs + e];
    y[(int64_t)s * ys + e] = act_f(v, kind, alpha);
    if (acc) acc[(int64_t)s * as + e] = v;
  }
}


__global__ void k_sparsify_finalize(const double* __restrict__ partials, int64_t n, double* norm_ema, double* kdev,
                                    double tp, double decay, int reset, int S) {
  pdl_wait();
  pdl_trigger();
  sparsify_finalize_all(partials, n, norm_ema, kdev, tp, decay, reset, blockIdx.x + 1, blockIdx.x);  // session = block
}

__global__ void k_sumsq(const float* __restrict__ x, int64_t xs, int64_t n, double* partials) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  double ss = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[(int64_t)s * xs + e];
    ss += v * v;
  }
  ss = block_sum<double>(ss, [](double v) { return warp_sum_d(v); });
  if (threadIdx.x == 0) partials[(int64_t)s * gridDim.x + blockIdx.x] = ss;
}

// ---------------------------------------------------------------------------
// inc_add / inc_mul (increment_ops.py:226-254)

__global__ void k_binary_dense(const float* __restrict__ a, int64_t as, const float* __restrict__ b, int64_t bs,
                               float* __restrict__ y, int64_t ys, int64_t n, int op) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float va = a[(int64_t)s * as + e], vb = b[(int64_t)s * bs + e];
    y[(int64_t)s * ys + e] = op ? __fmul_rn(va, vb) : __fadd_rn(va, vb);
  }
}


// upsample (increment_ops.py:271-285, tensors.py:259-282)
// ---------------------------------------------------------------------------

__global__ void k_upsample(TView in, TView out, int f, int mode) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t s_m[];  // proc | new (2 x GWo)
  const int i = blockIdx.x, c = blockIdx.y, s = blockIdx.z;
  const bool masked = in.f != nullptr;
  const int u0 = i * out.th, u1 = min(out.H, u0 + out.th);
  uint8_t* s_proc = s_m;
  uint8_t* s_new = s_m + out.GW;
  uint8_t* fo = masked ? out.fplane(s, c) + (int64_t)i * out.GW : nullptr;
  bool any = !masked;
  if (masked) {
    int rlo, rhi;
    if (mode == 0) {
      rlo = u0 / f;
      rhi = (u1 - 1) / f;
    } else {
      rlo = bilinear_tap(u0, in.H, f).i0;
      rhi = bilinear_tap(u1 - 1, in.H, f).i1;
    }
    const int alo = rlo / in.th, ahi = rhi / in.th;
    const uint8_t* F = in.fplane(s, c);
    for (int j = threadIdx.x; j < out.GW; j += blockDim.x) {
      const int v0 = j * out.tw, v1 = min(out.W, v0 + out.tw);
      int clo, chi;
      if (mode == 0) {
        clo = v0 / f;
        chi = (v1 - 1) / f;
      } else {
        clo = bilinear_tap(v0, in.W, f).i0;
        chi = bilinear_tap(v1 - 1, in.W, f).i1;
      }
      const int blo = clo / in.tw, bhi = chi / in.tw;
      uint8_t nf = 0;
      for (int a = alo; a <= ahi; ++a)
        for (int b = blo; b <= bhi; ++b) nf |= F[a * in.GW + b];
      nf = nf != 0;
      s_new[j] = nf;
      s_proc[j] = nf | fo[j];
      any |= s_proc[j] != 0;
    }
  }
  if (!__syncthreads_or(any)) return;
  const float* xv = in.plane(s, c);
  float* yv = out.plane(s, c);
  for (int v = threadIdx.x; v < out.W; v += blockDim.x) {
    if (masked && !s_proc[v / out.tw]) continue;
    if (mode == 0) {
      const int sx = v / f;
      for (int u = u0; u < u1; ++u) yv[(int64_t)u * out.W + v] = xv[(int64_t)(u / f) * in.W + sx];
    } else {
      const Tap tc = bilinear_tap(v, in.W, f);
      for (int u = u0; u < u1; ++u) {
        const Tap tr = bilinear_tap(u, in.H, f);
        const float* x0 = xv + (int64_t)tr.i0 * in.W;
        const float* x1 = xv + (int64_t)tr.i1 * in.W;
        const float ra = __fadd_rn(__fmul_rn(x0[tc.i0], tr.w0), __fmul_rn(x1[tc.i0], tr.w1));
        const float rb = __fadd_rn(__fmul_rn(x0[tc.i1], tr.w0), __fmul_rn(x1[tc.i1], tr.w1));
        yv[(int64_t)u * out.W + v] = __fadd_rn(__fmul_rn(ra, tc.w0), __fmul_rn(rb, tc.w1));
      }
    }
  }
  if (masked) {
    __syncthreads();
    for (int j = threadIdx.x; j < out.GW; j += blockDim.x) fo[j] = s_new[j];
  }
}

// ---------------------------------------------------------------------------
// maxpool (increment_ops.py:288-310, tensors.py:242-256)
// ---------------------------------------------------------------------------
// Does some pooling window of outputs [o0, o1) read a pixel of input tile a?
__device__ __forceinline__ bool pool_covers(int a, int o0, int o1, int st, int win, int tile) {
  for (int o = o0; o < o1; ++o) {
    const int lo = o * st, hi = lo + win - 1;
    if (lo / tile <= a && a <= hi / tile) return true;
  }
  return false;
}

__global__ void k_maxpool(TView in, const float* __restrict__ acc, int64_t as, TView out, int wh, int ww, int st) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t s_m[];
  const int i = blockIdx.x, c = blockIdx.y, s = blockIdx.z;
  const bool masked = in.f != nullptr;
  const int u0 = i * out.th, u1 = min(out.H, u0 + out.th);
  uint8_t* s_proc = s_m;
  uint8_t* s_new = s_m + out.GW;
  uint8_t* fo = masked ? out.fplane(s, c) + (int64_t)i * out.GW : nullptr;
  bool any = !masked;
  if (masked) {
    const int alo = (u0 * st) / in.th, ahi = ((u1 - 1) * st + wh - 1) / in.th;
    const uint8_t* F = in.fplane(s, c);
    for (int j = threadIdx.x; j < out.GW; j += blockDim.x) {
      const int v0 = j * out.tw, v1 = min(out.W, v0 + out.tw);
      const int blo = (v0 * st) / in.tw, bhi = ((v1 - 1) * st + ww - 1) / in.tw;
      uint8_t nf = 0;
      for (int a = alo; a <= ahi; ++a) {
        if (!pool_covers(a, u0, u1, st, wh, in.th)) continue;  // stride > window leaves gaps
        for (int b = blo; b <= bhi; ++b)
          if (pool_covers(b, v0, v1, st, ww, in.tw)) nf |= F[a * in.GW + b];
      }
      nf = nf != 0;
      s_new[j] = nf;
      s_proc[j] = nf | fo[j];
      any |= s_proc[j] != 0;
    }
  }
  if (!__syncthreads_or(any)) return;
  const float* xv = in.plane(s, c);
  const float* av = acc ? acc + (int64_t)s * as + (int64_t)c * in.H * in.W : nullptr;
  float* yv = out.plane(s, c);
  for (int v = threadIdx.x; v < out.W; v += blockDim.x) {
    if (masked && !s_proc[v / out.tw]) continue;
    for (int u = u0; u < u1; ++u) {
      float mb = -INFINITY, ma = -INFINITY;
      for (int r = 0; r < wh; ++r)
        for (int q = 0; q < ww; ++q) {
          const int64_t e = (int64_t)(u * st + r) * in.W + v * st + q;
          if (av) {
            const float a0 = av[e];
            mb = fmaxf(mb, a0);
            ma = fmaxf(ma, __fadd_rn(a0, xv[e]));
          } else {
            ma = fmaxf(ma, xv[e]);
          }
        }
      yv[(int64_t)u * out.W + v] = av ? __fsub_rn(ma, mb) : ma;
    }
  }
  if (masked) {
    __syncthreads();
    for (int j = threadIdx.x; j < out.GW; j += blockDim.x) fo[j] = s_new[j];
  }
}

static int bt(int W) { return W >= 192 ? 256 : (W >= 96 ? 128 : (W >= 48 ? 64 : 32)); }

static int dense_blocks(int64_t n) {
  int64_t b = cdiv64(n, 256 * 4);
  if (b > 2048) b = 2048;
  return (int)(b > 0 ? b : 1);
}


}  // namespace evc

using namespace evc;

extern "C" {

int evc_fold(const evc_tensor* dx, float* acc, int64_t acc_stride, int32_t S, void* stream);

int evc_act_dense(const float* x, int64_t xs, float* y, int64_t ys, float* acc, int64_t as, int64_t n, int32_t kind,
                  float alpha, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && y && S > 0, "act_dense: null argument");
  launch_pdl(k_act_dense, dim3(dim3(dense_blocks(n), S)), dim3(256), 0, as_stream(stream), x, xs, y, ys, acc, as, n, kind, alpha);
  EVC_LAUNCH_CHECK("act_dense");
  return EVC_OK;
}

int evc_sparsify_finalize(const double* partials, int64_t n, double* norm_ema, double* k, double tp, double decay,
                          int32_t reset, int32_t S, void* stream) {
  EVC_CHECK_ARG(partials && norm_ema && k && S > 0, "sparsify_finalize: null argument");
  launch_pdl(k_sparsify_finalize, dim3(S), dim3(256), 0, as_stream(stream), partials, n, norm_ema, k, tp, decay, reset, S);
  EVC_LAUNCH_CHECK("sparsify_finalize");
  return EVC_OK;
}

int evc_sumsq_dense(const float* x, int64_t xs, int64_t n, double* partials, int32_t n_blocks, int32_t S,
                    void* stream) {
  EVC_CHECK_ARG(x && partials && n_blocks > 0 && S > 0, "sumsq_dense: null argument");
  launch_pdl(k_sumsq, dim3(dim3(n_blocks, S)), dim3(256), 0, as_stream(stream), x, xs, n, partials);
  EVC_LAUNCH_CHECK("sumsq_dense");
  return EVC_OK;
}

int evc_binary_dense(const float* a, int64_t as, const float* b, int64_t bs, float* y, int64_t ys, int64_t n,
                     int32_t op, int32_t S, void* stream) {
  EVC_CHECK_ARG(a && b && y && S > 0, "binary_dense: null argument");
  launch_pdl(k_binary_dense, dim3(dim3(dense_blocks(n), S)), dim3(256), 0, as_stream(stream), a, as, b, bs, y, ys, n, op);
  EVC_LAUNCH_CHECK("binary_dense");
  return EVC_OK;
}

int evc_upsample(const evc_tensor* in, const evc_tensor* out, int32_t factor, int32_t mode, int32_t S,
                 void* stream) {
  EVC_CHECK_ARG(in && out && S > 0, "upsample: null argument");
  EVC_CHECK_ARG(factor == 2 || factor == 4, "upsample: factor must be 2 or 4");
  EVC_CHECK_ARG(mode == 0 || mode == 1, "upsample: unknown mode");
  EVC_CHECK_ARG((in->flags == nullptr) == (out->flags == nullptr), "upsample: masks on both or neither");
  TView vi = view_of(*in), vo = view_of(*out);
  launch_pdl(k_upsample, dim3(dim3(vo.GH, vo.C, S)), dim3(bt(vo.W)), 2 * vo.GW, as_stream(stream), vi, vo, factor, mode);
  EVC_LAUNCH_CHECK("upsample");
  return EVC_OK;
}

int evc_maxpool(const evc_tensor* in, float* acc, int64_t acc_stride, const evc_tensor* out, int32_t wh, int32_t ww,
                int32_t stride, int32_t S, void* stream) {
  EVC_CHECK_ARG(in && out && S > 0 && wh > 0 && ww > 0 && stride > 0, "maxpool: bad argument");
  EVC_CHECK_ARG((in->flags == nullptr) == (out->flags == nullptr), "maxpool: masks on both or neither");
  EVC_CHECK_ARG(!acc || in->flags, "maxpool: incremental mode needs masks");
  TView vi = view_of(*in), vo = view_of(*out);
  cudaStream_t st = as_stream(stream);
  launch_pdl(k_maxpool, dim3(dim3(vo.GH, vo.C, S)), dim3(bt(vo.W)), 2 * vo.GW, st, vi, acc, acc_stride, vo, wh, ww, stride);
  EVC_LAUNCH_CHECK("maxpool");
  if (acc) return evc_fold(in, acc, acc_stride, S, stream);  // AccState.fold (increment_ops.py:93-94)
  return EVC_OK;
}

}  // extern "C"

namespace evc {

// Byte fill of n segments in one launch (the dense refresh's resets: increment stores, flag grids,
// conv input shadows, region states -- 100+ memsets otherwise, most of them a few KB).  seg[i] =
// {address, bytes, value}; every CTA walks every segment with a grid-stride loop over its 16-byte
// aligned body (the unaligned head / tail bytes by the first CTA).
__global__ void __launch_bounds__(256) k_fill_segments(const evc_fill_segment* __restrict__ seg, int n) {
  pdl_wait();
  pdl_trigger();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < n; ++i) {
    uint8_t* p = reinterpret_cast<uint8_t*>(seg[i].addr);
    const int64_t nb = seg[i].bytes;
    const uint32_t b = seg[i].value & 0xffu, w = b * 0x01010101u;
    const int64_t head = std::min<int64_t>(nb, (int64_t)((16u - (reinterpret_cast<uintptr_t>(p) & 15u)) & 15u));
    const int64_t nv = (nb - head) >> 4, tail0 = head + (nv << 4);
    uint4* body = reinterpret_cast<uint4*>(p + head);
    const uint4 wv = make_uint4(w, w, w, w);
    for (int64_t e = tid; e < nv; e += nthr) body[e] = wv;
    if (blockIdx.x == 0) {
      for (int64_t e = threadIdx.x; e < head; e += blockDim.x) p[e] = (uint8_t)b;
      for (int64_t e = tail0 + threadIdx.x; e < nb; e += blockDim.x) p[e] = (uint8_t)b;
    }
  }
}

}  // namespace evc

extern "C" int evc_fill_segments(const evc_fill_segment* segs, int32_t n, int32_t n_blocks, void* stream) {
  EVC_CHECK_ARG(segs && n >= 0 && n_blocks > 0, "fill_segments: bad argument");
  if (n == 0) return EVC_OK;
  launch_pdl(evc::k_fill_segments, dim3(n_blocks), dim3(256), 0, evc::as_stream(stream), segs, (int)n);
  EVC_LAUNCH_CHECK("fill_segments");
  return EVC_OK;
}

namespace evc {
int init_elementwise() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_sumsq) != cudaSuccess) return EVC_ECUDA;
  const int rc = init_upsparsify();
  return rc ? rc : init_bands();
}
}  // namespace evc
