// Tiled elementwise increment kernels: inc_activation, sparsify_step, inc_add,
// inc_mul, integrate, masked copy, accumulator fold
// (increment_ops.py:226-254, sparsify.py:54-78, tensors.py:167-174).
//
// One CTA owns a "tile block": 32 channels x one tile row x a tile-aligned chunk
// of columns of one session (24 px for 6x6 tiles, a multiple of both the tile
// width and 4 so rows move as aligned float4s).  Tiles never straddle CTAs, so
// per-(channel, tile) flags live in shared memory; a float4 is processed when
// one of its tiles is live in an input OR was live in the output last step.
// Recomputing a dead element from all-zero inputs writes an exact zero, which
// keeps values under False flags at 0 (TileMask soundness, tensors.py:65-72),
// and every output flag is derived per element tile.  Float arithmetic uses _rn
// intrinsics so no FMA contraction changes the reference's float32 rounding.
//
// The sparsify op can also emit the channels-innermost shadow that the TMA
// conv GEMM reads (conv_fused.cu), staged through padded shared memory so the
// planar reads and the 128-byte channel runs are both coalesced.

#include <algorithm>

#include <cstdlib>

#include "common.cuh"

namespace evc {

constexpr int TB_C = 32;  // channels per tile block
constexpr int TB_THREADS = 256;
constexpr int TB_MAXJ = 32;  // max tiles per column chunk
constexpr int TB_UNROLL = 4;

struct TBGeo {
  int C, H, W, th, tw, GH, GW, CW, nCG, nJC, vec;
};

static int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }

static TBGeo tb_geo(const TView& v, bool aligned) {
  TBGeo g;
  g.C = v.C;
  g.H = v.H;
  g.W = v.W;
  g.th = v.th;
  g.tw = v.tw;
  g.GH = v.GH;
  g.GW = v.GW;
  const int l = v.tw / gcd_i(v.tw, 4) * 4;  // lcm(tw, 4)
  g.vec = (aligned && v.W % 4 == 0 && l <= 32) ? 4 : 1;
  const int unit = g.vec == 4 ? l : v.tw;
  g.CW = unit >= 32 ? unit : unit * (32 / unit);
  g.nCG = (v.C + TB_C - 1) / TB_C;
  g.nJC = (v.W + g.CW - 1) / g.CW;
  return g;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static bool al_view(const TView& v) {
  return !v.v || (al16(v.v) && v.vs % 4 == 0 && ((int64_t)v.H * v.W) % 4 == 0);
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

enum { OP_ACT = 0, OP_SPARSIFY = 1, OP_ADD = 2, OP_MUL = 3, OP_INTEGRATE = 4, OP_COPY = 5, OP_FOLD = 6, OP_ADD_ACT = 7 };

struct TBArgs {
  TView a, b, y;    // inputs (b optional) and output
  float* acc;       // activation / fold / mul-a accumulator, integrate target
  float* acc2;      // mul-b accumulator / sparsify residual
  int64_t as;       // accumulator session stride
  uint8_t* dlive;   // sparsify residual-live flags
  const double* k;  // sparsify k per session
  double* partials;
  double* norm_ema;
  double tp, decay;
  int* ticket;
  float* hwc;  // sparsify channels-innermost shadow (optional)
  int64_t hs;  // shadow session stride
  int cp;      // shadow channel stride
  int hp;      // shadow row pitch in pixels (padded width of the consumer conv's input)
  uint8_t* fany;  // sparsify: optional any-channel tile map of the output (OR-accumulated, zeroed per step)
  int write_chw;
  int pstride;     // sparsify: partial slots per session (evc_sparsify_partials; unused slots stay 0)
  int delta_zero;  // sparsify with tp == 0 and k == 0: the residual is identically 0, skip its traffic
  int kind;
  float alpha;
};

template <int V>
struct Vec;
template <>
struct Vec<4> {
  using T = float4;
  __device__ static T ld(const float* p) { return *reinterpret_cast<const float4*>(p); }
  __device__ static void st(float* p, const T& v) { *reinterpret_cast<float4*>(p) = v; }
  __device__ static float get(const T& v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w)); }
  __device__ static void set(T& v, int k, float x) {
    if (k == 0) v.x = x;
    else if (k == 1) v.y = x;
    else if (k == 2) v.z = x;
    else v.w = x;
  }
};
template <>
struct Vec<1> {
  using T = float;
  __device__ static T ld(const float* p) { return *p; }
  __device__ static void st(float* p, const T& v) { *p = v; }
  __device__ static float get(const T& v, int) { return v; }
  __device__ static void set(T& v, int, float x) { v = x; }
};

template <int OP, int V>
__global__ void __launch_bounds__(TB_THREADS) k_tiles(TBArgs p, TBGeo g) {
  pdl_wait();
  pdl_trigger();
  using VT = Vec<V>;
  using T = typename VT::T;
  __shared__ uint8_t s_proc[TB_C * TB_MAXJ];
  __shared__ uint8_t s_f1[TB_C * TB_MAXJ];  // sparsify: output value != 0
  __shared__ uint8_t s_f2[TB_C * TB_MAXJ];  // sparsify: residual != 0
  // sparsify shadow staging: [(row * 32 + col) * 33 + channel], padded -> conflict-free both ways
  __shared__ float s_y[(OP == OP_SPARSIFY) ? 8 * 32 * 33 : 1];
  const int jc = blockIdx.x % g.nJC;
  const int rest = blockIdx.x / g.nJC;
  const int cg = rest % g.nCG, i = rest / g.nCG;
  const int s = blockIdx.y;
  const int c0 = cg * TB_C, nc = min(TB_C, g.C - c0);
  const int x0 = jc * g.CW, ncol = min(g.W, x0 + g.CW) - x0;
  const int j0 = x0 / g.tw, nj = (ncol + g.tw - 1) / g.tw;
  const int r0 = i * g.th, nrow = min(g.H, r0 + g.th) - r0;

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
    } else {
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
  const bool stage = OP == OP_SPARSIFY && p.hwc && nrow <= 8 && ncol <= 32;
  if (active) {
    const int64_t HW = (int64_t)g.H * g.W;
    const double kd = OP == OP_SPARSIFY ? p.k[s] : 0.0;
    const bool use_k = kd > 0.0;
    const float k32 = __double2float_rn(kd);
    const int nq = ncol / V;  // vector units per row chunk (ncol % V == 0 by construction)
    const int n = nc * nrow * nq;
    const FDiv d_nq = fdiv_of(nq), d_nrow = fdiv_of(nrow), d_tw = fdiv_of(g.tw);
    const int64_t sa = (int64_t)s * p.a.vs, sy = (int64_t)s * p.y.vs, sacc = (int64_t)s * p.as;
    const int64_t sb = (OP == OP_ADD || OP == OP_MUL || OP == OP_ADD_ACT) ? (int64_t)s * p.b.vs : 0;
    for (int base = threadIdx.x; base < n; base += TB_THREADS * TB_UNROLL) {
      int64_t off[TB_UNROLL];
      int cl_[TB_UNROLL], r_[TB_UNROLL], xl_[TB_UNROLL];
      bool on[TB_UNROLL];
      T va[TB_UNROLL], vb[TB_UNROLL], vc[TB_UNROLL];
#pragma unroll
      for (int u = 0; u < TB_UNROLL; ++u) {
        const int e = base + u * TB_THREADS;
        on[u] = false;
        if (e >= n) continue;
        const int t2 = fdiv(e, d_nq), q = e - t2 * nq;
        const int cl = fdiv(t2, d_nrow), r = t2 - cl * nrow;
        const int xl = q * V;
        bool pr = false;
#pragma unroll
        for (int k = 0; k < V; ++k) pr |= s_proc[cl * nj + fdiv(xl + k, d_tw)] != 0;
        cl_[u] = cl;
        r_[u] = r;
        xl_[u] = xl;
        on[u] = pr;
        if (!pr) continue;
        off[u] = (int64_t)(c0 + cl) * HW + (int64_t)(r0 + r) * g.W + x0 + xl;
        va[u] = VT::ld(p.a.v + sa + off[u]);
        if (OP == OP_ADD || OP == OP_MUL || OP == OP_ADD_ACT) vb[u] = VT::ld(p.b.v + sb + off[u]);
        if (OP == OP_ACT || OP == OP_MUL || OP == OP_INTEGRATE || OP == OP_FOLD || OP == OP_ADD_ACT)
          vc[u] = VT::ld(p.acc + sacc + off[u]);
        if (OP == OP_SPARSIFY) {
          if (p.delta_zero) {
#pragma unroll
            for (int k = 0; k < V; ++k) VT::set(vc[u], k, 0.0f);
          } else {
            vc[u] = VT::ld(p.acc2 + sacc + off[u]);
          }
        }
        if (OP == OP_MUL) vb[u] = VT::ld(p.b.v + sb + off[u]);
      }
#pragma unroll
      for (int u = 0; u < TB_UNROLL; ++u) {
        const int e = base + u * TB_THREADS;
        if (e >= n) continue;
        if (!on[u]) {
          if (stage) {
#pragma unroll
            for (int k = 0; k < V; ++k) s_y[(r_[u] * 32 + xl_[u] + k) * 33 + cl_[u]] = 0.0f;
          }
          continue;
        }
        T out = va[u], acc_new = vc[u], acc2_new = vb[u];
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const float a = VT::get(va[u], k);
          if (OP == OP_ADD_ACT) {  // inc_add then inc_activation, the same float32 ops in order
            const float sm = __fadd_rn(a, VT::get(vb[u], k));
            const float a0 = VT::get(vc[u], k), a1 = __fadd_rn(a0, sm);
            VT::set(out, k, __fsub_rn(act_fn(a1, p.kind, p.alpha), act_fn(a0, p.kind, p.alpha)));
            VT::set(acc_new, k, a1);
          } else if (OP == OP_ACT) {
            const float a0 = VT::get(vc[u], k), a1 = __fadd_rn(a0, a);
            VT::set(out, k, __fsub_rn(act_fn(a1, p.kind, p.alpha), act_fn(a0, p.kind, p.alpha)));
            VT::set(acc_new, k, a1);
          } else if (OP == OP_SPARSIFY) {
            const float corr = __fadd_rn(VT::get(vc[u], k), a);
            float o, nd;
            if (use_k) {
              o = __fmul_rn(k32, floorf(__fadd_rn(0.5f, __fdiv_rn(corr, k32))));
              nd = __fsub_rn(corr, o);
            } else {
              o = corr;
              nd = 0.0f;
            }
            VT::set(out, k, o);
            VT::set(acc_new, k, nd);
            ss += (double)corr * (double)corr;
            const int ti = cl_[u] * nj + fdiv(xl_[u] + k, d_tw);
            if (o != 0.0f) s_f1[ti] = 1;
            if (nd != 0.0f) s_f2[ti] = 1;
            if (stage) s_y[(r_[u] * 32 + xl_[u] + k) * 33 + cl_[u]] = o;
          } else if (OP == OP_ADD) {
            VT::set(out, k, __fadd_rn(a, VT::get(vb[u], k)));
          } else if (OP == OP_MUL) {
            const float b = VT::get(vb[u], k);
            const float t1 = __fadd_rn(VT::get(vc[u], k), a);
            // acc_b lives in acc2; loaded below (kept scalar to limit registers)
            VT::set(acc_new, k, t1);
            VT::set(out, k, __fmul_rn(t1, b));
          } else if (OP == OP_INTEGRATE || OP == OP_FOLD) {
            VT::set(acc_new, k, __fadd_rn(VT::get(vc[u], k), a));
          }
        }
        if (OP == OP_MUL) {  // y = (acc_a + a) * b + acc_b * a ; acc_b += b
          float* pb2 = p.acc2 + sacc + off[u];
          T sbv = VT::ld(pb2);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const float a = VT::get(va[u], k), b = VT::get(vb[u], k), s2 = VT::get(sbv, k);
            VT::set(out, k, __fadd_rn(VT::get(out, k), __fmul_rn(s2, a)));
            VT::set(sbv, k, __fadd_rn(s2, b));
          }
          VT::st(pb2, sbv);
          (void)acc2_new;
        }
        if (OP == OP_ACT || OP == OP_ADD || OP == OP_MUL || OP == OP_COPY || OP == OP_ADD_ACT)
          VT::st(p.y.v + sy + off[u], out);
        if (OP == OP_SPARSIFY) {
          if (p.write_chw) VT::st(p.y.v + sy + off[u], out);
          if (p.hwc && !stage) {
#pragma unroll
            for (int k = 0; k < V; ++k)
              hwc_store(p.hwc + (int64_t)s * p.hs + ((int64_t)(r0 + r_[u]) * p.hp + x0 + xl_[u] + k) * hwc_px(p.cp), p.cp,
                        c0 + cl_[u], VT::get(out, k));
          }
          if (!p.delta_zero) VT::st(p.acc2 + sacc + off[u], acc_new);
        }
        if (OP == OP_ACT || OP == OP_MUL || OP == OP_INTEGRATE || OP == OP_FOLD || OP == OP_ADD_ACT)
          VT::st(p.acc + sacc + off[u], acc_new);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nc * nj; t += TB_THREADS) {
      const int cl = t / nj, jl = t % nj;
      const int64_t fo = ((int64_t)(c0 + cl) * g.GH + i) * g.GW + j0 + jl;
      if (OP == OP_ACT || OP == OP_COPY) {
        p.y.f[(int64_t)s * p.y.fs + fo] = p.a.f[(int64_t)s * p.a.fs + fo];
      } else if (OP == OP_SPARSIFY) {
        p.y.f[(int64_t)s * p.y.fs + fo] = s_f1[t];
        p.dlive[(int64_t)s * g.C * g.GH * g.GW + fo] = s_f2[t];
        if (p.fany && s_f1[t]) p.fany[((int64_t)s * g.GH + i) * g.GW + j0 + jl] = 1;  // benign race: all store 1
      } else if (OP == OP_ADD || OP == OP_MUL || OP == OP_ADD_ACT) {
        p.y.f[(int64_t)s * p.y.fs + fo] = p.a.f[(int64_t)s * p.a.fs + fo] | p.b.f[(int64_t)s * p.b.fs + fo];
      }
    }
    if (stage && (int)(threadIdx.x & 31) < nc) {  // lane = channel: 128-byte runs of heads and tails per pixel
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      float* dst = p.hwc + (int64_t)s * p.hs + (int64_t)r0 * p.hp * hwc_px(p.cp);
      for (int r = 0; r < nrow; ++r)
        for (int xl = warp; xl < ncol; xl += TB_THREADS / 32)
          hwc_store(dst + ((int64_t)r * p.hp + x0 + xl) * hwc_px(p.cp), p.cp, c0 + lane, s_y[(r * 32 + xl) * 33 + lane]);
    }
  }
  if (OP == OP_SPARSIFY) {
    const int nblocks = gridDim.x * gridDim.y;
    ss = block_sum<double>(ss, [](double v) { return warp_sum_d(v); });
    if (threadIdx.x == 0) p.partials[(int64_t)s * p.pstride + blockIdx.x] = ss;
    if (!p.ticket) return;  // norm / k folded later by evc_meter_step (one launch for every node)
    // last CTA to retire folds every session's partials into norm_ema / k (fixed order)
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(p.ticket, 1) == nblocks - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      sparsify_finalize_all(p.partials, p.pstride, p.norm_ema, const_cast<double*>(p.k), p.tp, p.decay, 0,
                            gridDim.y);
    }
  }
}

// integrate (tensors.py:167-174): y_run += where(live, dx, 0), flat over (session, channel,
// row, 4 columns): the output is small (C1: 2 x 256 x 256) so tile-row CTAs of 32 channels
// would leave most lanes idle; one float4 per thread, the tile flag read per vector.
__global__ void __launch_bounds__(256) k_integrate_flat(TView a, float* __restrict__ y, int64_t ys, int64_t nvec) {
  pdl_wait();
  pdl_trigger();
  const int W4 = a.W >> 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nvec; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t per_s = (int64_t)a.C * a.H * W4;
    const int s = (int)(e / per_s);
    const int64_t r = e - (int64_t)s * per_s;
    const int q = (int)(r % W4);
    const int64_t cu = r / W4;  // channel * H + row
    const int u = (int)(cu % a.H), c = (int)(cu / a.H);
    const int x = q * 4;
    const uint8_t* F = a.f + (int64_t)s * a.fs + ((int64_t)c * a.GH + u / a.th) * a.GW;
    const bool l0 = F[x / a.tw] != 0, l3 = F[(x + 3) / a.tw] != 0;
    if (!l0 && !l3 && F[(x + 1) / a.tw] == 0 && F[(x + 2) / a.tw] == 0) continue;
    const int64_t off = ((int64_t)c * a.H + u) * a.W + x;
    const float4 d = *reinterpret_cast<const float4*>(a.v + (int64_t)s * a.vs + off);
    float4* yp = reinterpret_cast<float4*>(y + (int64_t)s * ys + off);
    float4 v = *yp;
    if (F[x / a.tw]) v.x = __fadd_rn(v.x, d.x);
    if (F[(x + 1) / a.tw]) v.y = __fadd_rn(v.y, d.y);
    if (F[(x + 2) / a.tw]) v.z = __fadd_rn(v.z, d.z);
    if (F[(x + 3) / a.tw]) v.w = __fadd_rn(v.w, d.w);
    *yp = v;
  }
}

// t_p = 0 sparsify of a tensor with few channels (C <= 8, e.g. the 4-channel event input):
// one thread per pixel of a tile row x SM_TJ tiles, all channels per thread, so no lanes
// idle on missing channels.  y = 0 + x (sparsify.py:69-71); flags recomputed from the values
// (sparsify.py:77-78) through shared memory; the channels-innermost hi/lo shadow gets each
// pixel's C heads and C tails as contiguous runs.
constexpr int SM_TJ = 6, SM_RT = 4;  // tiles per CTA: SM_RT tile rows x SM_TJ tile columns
__global__ void __launch_bounds__(256) k_sparsify_small(TBArgs p) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint8_t s_f[SM_RT * 8 * SM_TJ];  // [tile row][channel][tile column]
  __shared__ double s_red[8];
  const TView& a = p.a;
  const int nJ = (a.GW + SM_TJ - 1) / SM_TJ;
  const int jb = blockIdx.x % nJ, ib = blockIdx.x / nJ, s = blockIdx.y;
  const int j0 = jb * SM_TJ, nj = min(SM_TJ, a.GW - j0);
  const int i0 = ib * SM_RT, ni = min(SM_RT, a.GH - i0);
  for (int t = threadIdx.x; t < SM_RT * 8 * SM_TJ; t += blockDim.x) s_f[t] = 0;
  __syncthreads();
  const int span = SM_TJ * a.tw, rows = ni * a.th;  // th, tw <= 6 (checked on host)
  const int64_t HW = (int64_t)a.H * a.W;
  const bool vec4 = a.C == 4 && (p.cp == 4 || p.cp == -4);  // 16-byte runs of heads and of tails per pixel
  float ss = 0.0f;
  for (int t = threadIdx.x; t < rows * span; t += blockDim.x) {
    const int r = t / span, xq = t - r * span;
    const int u = i0 * a.th + r, x = j0 * a.tw + xq;
    if (u >= a.H || xq >= nj * a.tw || x >= a.W) continue;
    const int64_t off = (int64_t)u * a.W + x;
    const float* src = a.v + (int64_t)s * a.vs + off;
    float v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < a.C) v[c] = __fadd_rn(0.0f, src[c * HW]);
    uint8_t* f = s_f + (r / a.th) * 8 * SM_TJ + xq / a.tw;
    float* sh = p.hwc ? p.hwc + (int64_t)s * p.hs + ((int64_t)u * p.hp + x) * hwc_px(p.cp) : nullptr;
    if (sh && vec4 && p.cp < 0) {
      *reinterpret_cast<float4*>(sh) = make_float4(v[0], v[1], v[2], v[3]);
    } else if (sh && vec4) {
      const float4 h = make_float4(tf32_head(v[0]), tf32_head(v[1]), tf32_head(v[2]), tf32_head(v[3]));
      *reinterpret_cast<float4*>(sh) = h;
      *reinterpret_cast<float4*>(sh + 4) =
          make_float4(__fsub_rn(v[0], h.x), __fsub_rn(v[1], h.y), __fsub_rn(v[2], h.z), __fsub_rn(v[3], h.w));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c >= a.C) break;
      if (p.write_chw) p.y.v[(int64_t)s * p.y.vs + c * HW + off] = v[c];
      if (sh && !vec4) hwc_store(sh, p.cp, c, v[c]);
      ss = __fmaf_rn(v[c], v[c], ss);
      if (v[c] != 0.0f) f[c * SM_TJ] = 1;
    }
  }
  double d = warp_sum_d((double)ss);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = d;
  __syncthreads();
  for (int t = threadIdx.x; t < ni * a.C * nj; t += blockDim.x) {
    const int il = t / (a.C * nj), e = t - il * a.C * nj, c = e / nj, jl = e - c * nj;
    const int64_t fo = ((int64_t)c * a.GH + i0 + il) * a.GW + j0 + jl;
    p.y.f[(int64_t)s * p.y.fs + fo] = s_f[(il * 8 + c) * SM_TJ + jl];
  }
  if (p.fany && threadIdx.x < ni * nj) {
    const int il = threadIdx.x / nj, jl = threadIdx.x - il * nj;
    int any = 0;
    for (int c = 0; c < a.C; ++c) any |= s_f[(il * 8 + c) * SM_TJ + jl];
    if (any) p.fany[((int64_t)s * a.GH + i0 + il) * a.GW + j0 + jl] = 1;
  }
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
    p.partials[(int64_t)s * p.pstride + blockIdx.x] = t;
  }
}

static bool small_ok(const TView& v) { return v.C <= 8 && v.th <= 6 && v.tw <= 6; }
static int small_blocks(const TView& v) { return ((v.GH + SM_RT - 1) / SM_RT) * ((v.GW + SM_TJ - 1) / SM_TJ); }

template <int OP>
static void launch_op(const TBArgs& p, const TBGeo& g, int S, cudaStream_t st) {
  dim3 grid((unsigned)(g.GH * g.nCG * g.nJC), (unsigned)S);
  if (g.vec == 4)
    launch_pdl(k_tiles<OP, 4>, dim3(grid), dim3(TB_THREADS), 0, st, p, g);
  else
    launch_pdl(k_tiles<OP, 1>, dim3(grid), dim3(TB_THREADS), 0, st, p, g);
}

static int tb_launch(int op, const TBArgs& p, int S, cudaStream_t st) {
  bool al = al_view(p.a) && al_view(p.y) && al_view(p.b);
  if (p.acc) al = al && al16(p.acc) && p.as % 4 == 0;
  if (p.acc2) al = al && al16(p.acc2) && p.as % 4 == 0;
  const TBGeo g = tb_geo(p.a, al);
  switch (op) {
    case OP_ACT: launch_op<OP_ACT>(p, g, S, st); break;
    case OP_SPARSIFY: launch_op<OP_SPARSIFY>(p, g, S, st); break;
    case OP_ADD: launch_op<OP_ADD>(p, g, S, st); break;
    case OP_MUL: launch_op<OP_MUL>(p, g, S, st); break;
    case OP_INTEGRATE: launch_op<OP_INTEGRATE>(p, g, S, st); break;
    case OP_COPY: launch_op<OP_COPY>(p, g, S, st); break;
    case OP_FOLD: launch_op<OP_FOLD>(p, g, S, st); break;
    case OP_ADD_ACT: launch_op<OP_ADD_ACT>(p, g, S, st); break;
    default: return EVC_EINVAL;
  }
  return EVC_OK;
}

int init_bands() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, k_tiles<OP_SPARSIFY, 4>) == cudaSuccess ? EVC_OK : EVC_ECUDA;
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
  const int rc = tb_launch(OP_ACT, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("act_delta");
  return rc;
}

int64_t evc_sparsify_partials(const evc_tensor* dx) {
  if (!dx) return -1;
  const TView v = view_of(*dx);
  const TBGeo g = tb_geo(v, true);
  const TBGeo g1 = tb_geo(v, false);
  return std::max(std::max(g.GH * g.nCG * g.nJC, g1.GH * g1.nCG * g1.nJC), small_ok(v) ? small_blocks(v) : 0);
}

int evc_sparsify(const evc_tensor* dx, float* delta, int64_t ds, uint8_t* dlive, const evc_tensor* y, double* k,
                 double* norm_ema, double tp, double ema_decay, double* partials, int32_t* ticket, float* hwc,
                 int32_t cp, int64_t hwc_stride, int32_t hwc_pitch, uint8_t* fany, int32_t write_chw,
                 int32_t delta_zero, int32_t S, void* stream) {
  EVC_CHECK_ARG(dx && y && delta && dlive && k && norm_ema && partials && dx->flags && y->flags && S > 0,
                "sparsify: null argument");
  EVC_CHECK_ARG(write_chw || hwc, "sparsify: no output requested");
  EVC_CHECK_ARG(!hwc || (std::abs(cp) >= dx->C && cp % 4 == 0 && hwc_pitch >= dx->W),
                "sparsify: shadow channel count must cover C (multiple of 32), pitch >= W");
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
  p.hp = hwc_pitch;
  p.cp = cp;
  p.fany = fany;
  p.write_chw = write_chw;
  p.delta_zero = delta_zero;
  p.pstride = (int)evc_sparsify_partials(dx);
  if (delta_zero && !ticket && small_ok(p.a)) {  // few channels at t_p = 0: thread per pixel
    launch_pdl(k_sparsify_small, dim3((unsigned)small_blocks(p.a), (unsigned)S), dim3(256), 0, as_stream(stream), p);
    EVC_LAUNCH_CHECK("sparsify_small");
    return EVC_OK;
  }
  const int rc = tb_launch(OP_SPARSIFY, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("sparsify");
  return rc;
}

int evc_add(const evc_tensor* a, const evc_tensor* b, const evc_tensor* y, int32_t S, void* stream) {
  EVC_CHECK_ARG(a && b && y && a->flags && b->flags && y->flags && S > 0, "add: null argument");
  TBArgs p = {};
  p.a = view_of(*a);
  p.b = view_of(*b);
  p.y = view_of(*y);
  const int rc = tb_launch(OP_ADD, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("add");
  return rc;
}

int evc_add_act(const evc_tensor* a, const evc_tensor* b, float* acc, int64_t acc_stride, const evc_tensor* y,
                int32_t kind, float alpha, int32_t S, void* stream) {
  EVC_CHECK_ARG(a && b && y && acc && a->flags && b->flags && y->flags && S > 0 && kind >= 0 && kind <= 3,
                "add_act: bad argument");
  TBArgs p = {};
  p.a = view_of(*a);
  p.b = view_of(*b);
  p.y = view_of(*y);
  p.acc = acc;
  p.as = acc_stride;
  p.kind = kind;
  p.alpha = alpha;
  const int rc = tb_launch(OP_ADD_ACT, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("add_act");
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
  const int rc = tb_launch(OP_MUL, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("mul");
  return rc;
}

int evc_integrate(float* y_run, int64_t y_stride, const evc_tensor* dx, int32_t S, void* stream) {
  EVC_CHECK_ARG(y_run && dx && dx->vals && dx->flags && S > 0, "integrate: null argument");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.acc = y_run;
  p.as = y_stride;
  if (p.a.W % 4 == 0 && al16(p.a.v) && al16(y_run) && p.a.vs % 4 == 0 && y_stride % 4 == 0) {
    const int64_t nvec = (int64_t)S * p.a.C * p.a.H * (p.a.W / 4);
    const int grid = (int)std::min<int64_t>((nvec + 255) / 256, 148 * 16);
    launch_pdl(k_integrate_flat, dim3(grid), dim3(256), 0, as_stream(stream), p.a, y_run, y_stride, nvec);
    EVC_LAUNCH_CHECK("integrate");
    return EVC_OK;
  }
  const int rc = tb_launch(OP_INTEGRATE, p, S, as_stream(stream));
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
  const int rc = tb_launch(OP_COPY, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("copy_masked");
  return rc;
}

int evc_fold(const evc_tensor* dx, float* acc, int64_t acc_stride, int32_t S, void* stream) {
  EVC_CHECK_ARG(dx && dx->flags && acc && S > 0, "fold: null argument");
  TBArgs p = {};
  p.a = view_of(*dx);
  p.acc = acc;
  p.as = acc_stride;
  const int rc = tb_launch(OP_FOLD, p, S, as_stream(stream));
  EVC_LAUNCH_CHECK("fold");
  return rc;
}

}  // extern "C"
