// Tiled elementwise increment kernels: inc_activation, sparsify_step, inc_add,
// inc_mul, integrate, masked copy, accumulator fold
// (increment_ops.py:226-254, sparsify.py:54-78, tensors.py:167-174).
//
// One CTA owns a "tile block": 32 channels x one tile row x a tile-aligned chunk
// of columns (CW = tw * floor(32 / tw) pixels) of one session.  Tiles never
// straddle CTAs, so per-(channel, tile) flags live in shared memory; a tile is
// processed when it is live in an input OR was live in the output last step
// (recomputing a previously-live tile from all-zero inputs writes exact zeros,
// which keeps values under False flags at 0 -- TileMask soundness,
// tensors.py:65-72).  Float arithmetic uses _rn intrinsics so no FMA
// contraction changes the reference's float32 rounding sequence.
//
// The sparsify op can also emit the channels-innermost shadow that the TMA
// conv GEMM reads (conv_tma.cu), staged through shared memory so both the
// planar reads and the 128-byte channel runs are coalesced.

#include "common.cuh"

namespace evc {

constexpr int TB_C = 32;        // channels per tile block
constexpr int TB_THREADS = 256;
constexpr int TB_MAXJ = 32;     // max tiles per column chunk

struct TBGeo {
  int C, H, W, th, tw, GH, GW, CW, nCG, nJC;
};

static TBGeo tb_geo(const TView& v) {
  TBGeo g;
  g.C = v.C;
  g.H = v.H;
  g.W = v.W;
  g.th = v.th;
  g.tw = v.tw;
  g.GH = v.GH;
  g.GW = v.GW;
  g.CW = v.tw >= 32 ? v.tw : v.tw * (32 / v.tw);
  g.nCG = (v.C + TB_C - 1) / TB_C;
  g.nJC = (v.W + g.CW - 1) / g.CW;
  return g;
}

__device__ __forceinline__ float act_fn(float x, int kind, float alpha) {
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

enum { OP_ACT = 0, OP_SPARSIFY = 1, OP_ADD = 2, OP_MUL = 3, OP_INTEGRATE = 4, OP_COPY = 5, OP_FOLD = 6 };

struct TBArgs {
  TView a, b, y;       // inputs (b optional) and output
  float* acc;          // activation / fold / mul-a accumulator, integrate target
  float* acc2;         // mul-b accumulator / sparsify residual
  int64_t as;          // accumulator session stride
  uint8_t* dlive;      // sparsify residual-live flags
  const double* k;     // sparsify k per session
  double* partials;    // sparsify sum(corrected^2) per tile block
  double* norm_ema;
  double tp, decay;
  int* ticket;
  float* hwc;          // sparsify channels-innermost shadow (optional)
  int64_t hs;          // shadow session stride
  int cp;              // shadow channel stride
  int write_chw;       // sparsify: also write the planar output
  int kind;            // activation kind
  float alpha;
};



template <int OP>
__global__ void __launch_bounds__(TB_THREADS) k_tiles(TBArgs p, TBGeo g) {
  __shared__ uint8_t s_proc[TB_C * TB_MAXJ];
  __shared__ uint8_t s_f1[TB_C * TB_MAXJ];  // output flag (values != 0) / residual-live
  __shared__ uint8_t s_f2[TB_C * TB_MAXJ];
  __shared__ float s_y[(OP == OP_SPARSIFY) ? TB_C * 8 * 32 : 1];  // staged outputs for the shadow
  const int jc = blockIdx.x % g.nJC;
  const int rest = blockIdx.x / g.nJC;
  const int cg = rest % g.nCG, i = rest / g.nCG;
  const int s = blockIdx.y;
  const int c0 = cg * TB_C, nc = min(TB_C, g.C - c0);
  const int x0 = jc * g.CW, x1 = min(g.W, x0 + g.CW), ncol = x1 - x0;
  const int j0 = x0 / g.tw, nj = (ncol + g.tw - 1) / g.tw;
  const int r0 = i * g.th, nrow = min(g.H, r0 + g.th) - r0;

  // ---- per-(channel, tile) processing decision
  bool any = false;
  for (int t = threadIdx.x; t < nc * nj; t += TB_THREADS) {
    const int cl = t / nj, jl = t % nj;
    const int64_t fo = ((int64_t)(c0 + cl) * g.GH + i) * g.GW + j0 + jl;
    uint8_t pr;
    if (OP == OP_ACT || OP == OP_INTEGRATE || OP == OP_FOLD) {
      pr = p.a.f[(int64_t)s * p.a.fs + fo];
      if (OP == OP_ACT) pr |= p.y.f[(int64_t)s * p.y.fs + fo];
    } else if (OP == OP_SPARSIFY) {
      pr = p.a.f[(int64_t)s * p.a.fs + fo] | p.y.f[(int64_t)s * p.y.fs + fo] |
           p.dlive[(int64_t)s * g.C * g.GH * g.GW + fo];
    } else if (OP == OP_COPY) {
      pr = p.a.f[(int64_t)s * p.a.fs + fo] | p.y.f[(int64_t)s * p.y.fs + fo];
    } else {  // add / mul
      pr = p.a.f[(int64_t)s * p.a.fs + fo] | p.b.f[(int64_t)s * p.b.fs + fo] | p.y.f[(int64_t)s * p.y.fs + fo];
    }
    s_proc[t] = pr != 0;
    s_f1[t] = 0;
    s_f2[t] = 0;
    any |= pr != 0;
  }
  double ss = 0.0;
  const bool active = __syncthreads_or(any) != 0;
  if (OP != OP_SPARSIFY && !active) return;
  // stage sparsify outputs for the shadow when the block fits (th <= 8, CW <= 32)
  const bool stage = OP == OP_SPARSIFY && p.hwc && nrow <= 8 && ncol <= 32;
  if (active) {
    const int64_t HW = (int64_t)g.H * g.W;
    const double kd = OP == OP_SPARSIFY ? p.k[s] : 0.0;
    const bool use_k = kd > 0.0;
    const float k32 = __double2float_rn(kd);
    const int n = nc * nrow * ncol;
    for (int e = threadIdx.x; e < n; e += TB_THREADS) {
      const int xl = e % ncol, t2 = e / ncol;
      const int r = t2 % nrow, cl = t2 / nrow;
      const int ti = cl * nj + xl / g.tw;
      if (!s_proc[ti]) {
        if (stage) s_y[(cl * nrow + r) * 32 + xl] = 0.0f;
        continue;
      }
      const int c = c0 + cl;
      const int64_t off = (int64_t)c * HW + (int64_t)(r0 + r) * g.W + x0 + xl;
      if (OP == OP_ACT) {
        float* av = p.acc + (int64_t)s * p.as + off;
        const float a0 = *av, a1 = __fadd_rn(a0, p.a.v[(int64_t)s * p.a.vs + off]);
        p.y.v[(int64_t)s * p.y.vs + off] = __fsub_rn(act_fn(a1, p.kind, p.alpha), act_fn(a0, p.kind, p.alpha));
        *av = a1;
      } else if (OP == OP_SPARSIFY) {
        float* dl = p.acc2 + (int64_t)s * p.as + off;
        const float corr = __fadd_rn(*dl, p.a.v[(int64_t)s * p.a.vs + off]);
        float out, nd;
        if (use_k) {
          out = __fmul_rn(k32, floorf(__fadd_rn(0.5f, __fdiv_rn(corr, k32))));
          nd = __fsub_rn(corr, out);
        } else {
          out = corr;
          nd = 0.0f;
        }
        if (p.write_chw) p.y.v[(int64_t)s * p.y.vs + off] = out;
        if (stage) {
          s_y[(cl * nrow + r) * 32 + xl] = out;
        } else if (p.hwc) {
          p.hwc[(int64_t)s * p.hs + ((int64_t)(r0 + r) * g.W + x0 + xl) * p.cp + c] = out;
        }
        *dl = nd;
        ss += (double)corr * (double)corr;
        if (out != 0.0f) s_f1[ti] = 1;
        if (nd != 0.0f) s_f2[ti] = 1;
      } else if (OP == OP_ADD || OP == OP_MUL) {
        const float va = p.a.v[(int64_t)s * p.a.vs + off], vb = p.b.v[(int64_t)s * p.b.vs + off];
        if (OP == OP_ADD) {
          p.y.v[(int64_t)s * p.y.vs + off] = __fadd_rn(va, vb);
        } else {
          float* sa = p.acc + (int64_t)s * p.as + off;
          float* sb = p.acc2 + (int64_t)s * p.as + off;
          const float t1 = __fadd_rn(*sa, va);
          p.y.v[(int64_t)s * p.y.vs + off] = __fadd_rn(__fmul_rn(t1, vb), __fmul_rn(*sb, va));
          *sa = t1;
          *sb = __fadd_rn(*sb, vb);
        }
      } else if (OP == OP_INTEGRATE || OP == OP_FOLD) {
        float* yv = p.acc + (int64_t)s * p.as + off;
        *yv = __fadd_rn(*yv, p.a.v[(int64_t)s * p.a.vs + off]);
      } else if (OP == OP_COPY) {
        p.y.v[(int64_t)s * p.y.vs + off] = p.a.v[(int64_t)s * p.a.vs + off];
      }
    }
    __syncthreads();
    // ---- output flags
    for (int t = threadIdx.x; t < nc * nj; t += TB_THREADS) {
      const int cl = t / nj, jl = t % nj;
      const int64_t fo = ((int64_t)(c0 + cl) * g.GH + i) * g.GW + j0 + jl;
      if (OP == OP_ACT || OP == OP_COPY) {
        p.y.f[(int64_t)s * p.y.fs + fo] = p.a.f[(int64_t)s * p.a.fs + fo];
      } else if (OP == OP_SPARSIFY) {
        p.y.f[(int64_t)s * p.y.fs + fo] = s_f1[t];
        p.dlive[(int64_t)s * g.C * g.GH * g.GW + fo] = s_f2[t];
      } else if (OP == OP_ADD || OP == OP_MUL) {
        p.y.f[(int64_t)s * p.y.fs + fo] = p.a.f[(int64_t)s * p.a.fs + fo] | p.b.f[(int64_t)s * p.b.fs + fo];
      }
    }
    if (stage) {  // channels-innermost shadow: 32-channel runs per pixel
      float* dst = p.hwc + (int64_t)s * p.hs;
      for (int e = threadIdx.x; e < nrow * ncol * TB_C; e += TB_THREADS) {
        const int cl = e % TB_C, pix = e / TB_C;
        if (cl >= nc) continue;
        const int r = pix / ncol, xl = pix % ncol;
        dst[((int64_t)(r0 + r) * g.W + x0 + xl) * p.cp + c0 + cl] = s_y[(cl * nrow + r) * 32 + xl];
      }
    }
  }
  if (OP == OP_SPARSIFY) {
    const int nblocks = gridDim.x * gridDim.y;
    ss = block_sum<double>(ss, [](double v) { return warp_sum_d(v); });
    if (threadIdx.x == 0) p.partials[(int64_t)s * gridDim.x + blockIdx.x] = ss;
    // last CTA to retire folds every session's partials into norm_ema / k
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(p.ticket, 1) == nblocks - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      sparsify_finalize_all(p.partials, gridDim.x, p.norm_ema, const_cast<double*>(p.k), p.tp, p.decay, 0,
                            gridDim.y);
    }
  }
}

static int tb_launch(int op, const TBArgs& p, const TBGeo& g, int S, cudaStream_t st) {
  dim3 grid((unsigned)(g.GH * g.nCG * g.nJC), (unsigned)S);
  switch (op) {
    case OP_ACT: k_tiles<OP_ACT><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_SPARSIFY: k_tiles<OP_SPARSIFY><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_ADD: k_tiles<OP_ADD><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_MUL: k_tiles<OP_MUL><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_INTEGRATE: k_tiles<OP_INTEGRATE><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_COPY: k_tiles<OP_COPY><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    case OP_FOLD: k_tiles<OP_FOLD><<<grid, TB_THREADS, 0, st>>>(p, g); break;
    default: return EVC_EINVAL;
  }
  return EVC_OK;
}

int tiles_partials(const evc_tensor* t) {
  const TBGeo g = tb_geo(view_of(*t));
  return g.GH * g.nCG * g.nJC;
}

int init_bands() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, k_tiles<OP_SPARSIFY>) == cudaSuccess ? EVC_OK : EVC_ECUDA;
}

}  // namespace evc

using namespace evc;

extern "C" {

int evc_act_delta(const evc_tensor* dx, float* acc, int64_t acc_stride, const evc_tensor* y, int32_t kind,
                  float alpha, int32_t S, void* stream) {
  EVC_CHECK_ARG(dx && y && acc && dx->flags && y->flags && S > 0, "act_delta: null argument");
  EVC_CHECK_ARG(kind >= 0 && kind <= 3, "act_delta: unknown activation");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.y = view_of(*y);
  p.acc = acc;
  p.as = acc_stride;
  p.kind = kind;
  p.alpha = alpha;
  const int rc = tb_launch(OP_ACT, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("act_delta");
  return rc;
}

int64_t evc_sparsify_partials(const evc_tensor* dx) { return dx ? tiles_partials(dx) : -1; }

int evc_sparsify(const evc_tensor* dx, float* delta, int64_t ds, uint8_t* dlive, const evc_tensor* y, double* k,
                 double* norm_ema, double tp, double ema_decay, double* partials, int32_t* ticket, float* hwc,
                 int32_t cp, int64_t hwc_stride, int32_t write_chw, int32_t S, void* stream) {
  EVC_CHECK_ARG(dx && y && delta && dlive && k && norm_ema && partials && ticket && dx->flags && y->flags && S > 0,
                "sparsify: null argument");
  EVC_CHECK_ARG(write_chw || hwc, "sparsify: no output requested");
  EVC_CHECK_ARG(!hwc || cp >= dx->C, "sparsify: shadow channel stride too small");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.y = view_of(*y);
  p.acc2 = delta;
  p.as = ds;
  p.dlive = dlive;
  p.k = k;
  p.partials = partials;
  p.norm_ema = norm_ema;
  p.tp = tp;
  p.decay = ema_decay;
  p.ticket = ticket;
  p.hwc = hwc;
  p.hs = hwc_stride;
  p.cp = cp;
  p.write_chw = write_chw;
  const int rc = tb_launch(OP_SPARSIFY, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("sparsify");
  return rc;
}

int evc_add(const evc_tensor* a, const evc_tensor* b, const evc_tensor* y, int32_t S, void* stream) {
  EVC_CHECK_ARG(a && b && y && a->flags && b->flags && y->flags && S > 0, "add: null argument");
  TBArgs p = {};
  p.a = view_of(*a);
  p.b = view_of(*b);
  p.y = view_of(*y);
  const int rc = tb_launch(OP_ADD, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("add");
  return rc;
}

int evc_mul(const evc_tensor* a, const evc_tensor* b, float* acc_a, float* acc_b, int64_t acc_stride,
            const evc_tensor* y, int32_t S, void* stream) {
  EVC_CHECK_ARG(a && b && y && acc_a && acc_b && a->flags && b->flags && y->flags && S > 0, "mul: null argument");
  TBArgs p = {};
  p.a = view_of(*a);
  p.b = view_of(*b);
  p.y = view_of(*y);
  p.acc = acc_a;
  p.acc2 = acc_b;
  p.as = acc_stride;
  const int rc = tb_launch(OP_MUL, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("mul");
  return rc;
}

int evc_integrate(float* y_run, int64_t y_stride, const evc_tensor* dx, int32_t S, void* stream) {
  EVC_CHECK_ARG(y_run && dx && dx->vals && dx->flags && S > 0, "integrate: null argument");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.acc = y_run;
  p.as = y_stride;
  const int rc = tb_launch(OP_INTEGRATE, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("integrate");
  return rc;
}

int evc_copy_masked(const evc_tensor* src, const evc_tensor* dst, int32_t S, void* stream) {
  EVC_CHECK_ARG(src && dst && src->flags && dst->flags && S > 0, "copy_masked: null argument");
  TBArgs p = {};
  p.a = view_of(*src);
  p.y = view_of(*dst);
  EVC_CHECK_ARG(p.a.C == p.y.C && p.a.H == p.y.H && p.a.W == p.y.W && p.a.th == p.y.th && p.a.tw == p.y.tw,
                "copy_masked: shape");
  const int rc = tb_launch(OP_COPY, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("copy_masked");
  return rc;
}

int evc_fold(const evc_tensor* dx, float* acc, int64_t acc_stride, int32_t S, void* stream) {
  EVC_CHECK_ARG(dx && dx->flags && acc && S > 0, "fold: null argument");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.acc = acc;
  p.as = acc_stride;
  const int rc = tb_launch(OP_FOLD, p, tb_geo(p.a), S, as_stream(stream));
  EVC_LAUNCH_CHECK("fold");
  return rc;
}

}  // extern "C"
