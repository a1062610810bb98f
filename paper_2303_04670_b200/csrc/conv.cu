// Incremental convolution: mask propagation + exact FLOP meter, and the
// gather -> GEMM -> scatter over active output tiles.
//
// Reference: inc_conv2d (increment_ops.py:126-194), dense_conv2d
// (tensors.py:205-228).  Values of the incremental conv equal the bias-free
// convolution of the increment: the reference's per-channel skip only drops
// taps that read exact zeros (mask soundness), so computing every channel at
// every site of an active output tile gives the same sum (up to float
// reassociation) and exact zeros at the sites the reference skips.
//
// Masks and the meter are computed from the input tile flags only:
//   out tile (i,j) live  <=>  some site (u,v) in it has a tap on a live tile
//   performed = 2*C_out * sum_c sum_{(u,v): L_c>0} (K^2 - inb(u,v) + L_c(u,v))
// with L_c(u,v) the live in-bounds taps of channel c and inb the in-bounds
// taps (increment_ops.py:165-191; padding taps count, dead in-bounds taps do
// not), plus the all-false / all-true shortcuts (increment_ops.py:148-154).

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace evc {

// ---------------------------------------------------------------------------
// static per-layer table
// ---------------------------------------------------------------------------
// [0..7]   header: Ho, Wo, kh, kw, K, rows_off, cols_off, kdec_off
// rows:    Ho x (3 + kh): a_first, n_a, inR, cnt[kh]
// cols:    Wo x (3 + kw): b_first, n_b, inC, cnt[kw]
// kdec:    K x 2: c*H*W + r*W + q,  (r << 16) | q      (k = (c*kh + r)*kw + q)
struct TabHdr {
  int Ho, Wo, kh, kw, K, rows, cols, kdec;
};

static void axis_table(int n_out, int n_in, int k, int stride, int pad, int tile, int32_t* dst) {
  const int rec = 3 + k;
  for (int u = 0; u < n_out; ++u) {
    int32_t* e = dst + (int64_t)u * rec;
    for (int q = 0; q < rec; ++q) e[q] = 0;
    int first = -1, inb = 0;
    for (int r = 0; r < k; ++r) {
      const int y = u * stride - pad + r;
      if (y < 0 || y >= n_in) continue;
      const int a = y / tile;
      if (first < 0) first = a;
      e[3 + (a - first)] += 1;
      ++inb;
    }
    int n = 0;
    for (int q = 0; q < k; ++q)
      if (e[3 + q]) n = q + 1;
    e[0] = first < 0 ? 0 : first;
    e[1] = n;
    e[2] = inb;
  }
}

// ---------------------------------------------------------------------------
// mask propagation + meter   (one CTA per (output tile, session))
// ---------------------------------------------------------------------------
struct MaskArgs {
  TView in, out;
  const int32_t* tab;
  const int32_t* in_true;
  uint8_t* tile_active;
  int64_t* meter;
  int c_in, c_out, kk;
};

__global__ void __launch_bounds__(128) k_conv_mask(MaskArgs a) {
  const int t = blockIdx.x, s = blockIdx.y;
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int GWo = a.out.GW, T = a.out.GH * a.out.GW;
  const int i = t / GWo, j = t % GWo;
  const int u0 = i * a.out.th, u1 = min(h.Ho, u0 + a.out.th);
  const int v0 = j * a.out.tw, v1 = min(h.Wo, v0 + a.out.tw);
  const int32_t* rows = a.tab + h.rows;
  const int32_t* cols = a.tab + h.cols;
  const int rrec = 3 + h.kh, crec = 3 + h.kw;

  const int64_t total_in = (int64_t)a.c_in * a.in.GH * a.in.GW;
  const int cnt = a.in_true[s];
  long long contrib = 0;  // sum_c sum_sites (kk - inb + L)  (before the 2*C_out factor)
  if (cnt == 0) {
    contrib = 0;
  } else if ((int64_t)cnt == total_in) {
    contrib = (long long)a.kk * a.c_in * (u1 - u0) * (v1 - v0);  // dense shortcut
  } else {
    // input tile box touched by this output tile
    int A0 = INT32_MAX, A1 = -1, B0 = INT32_MAX, B1 = -1, nr = 0, nc = 0;
    for (int u = u0; u < u1; ++u) {
      const int32_t* e = rows + (int64_t)u * rrec;
      if (e[1]) { A0 = min(A0, e[0]); A1 = max(A1, e[0] + e[1] - 1); }
      nr += e[2] > 0;
    }
    for (int v = v0; v < v1; ++v) {
      const int32_t* e = cols + (int64_t)v * crec;
      if (e[1]) { B0 = min(B0, e[0]); B1 = max(B1, e[0] + e[1] - 1); }
      nc += e[2] > 0;
    }
    const long long all_live = (long long)a.kk * nr * nc;
    long long acc = 0;
    if (A1 >= 0 && B1 >= 0) {
      for (int c = threadIdx.x; c < a.c_in; c += blockDim.x) {
        const uint8_t* F = a.in.fplane(s, c);
        int any = 0, all = 1;
        for (int aa = A0; aa <= A1; ++aa)
          for (int bb = B0; bb <= B1; ++bb) {
            const int f = F[aa * a.in.GW + bb] != 0;
            any |= f;
            all &= f;
          }
        if (!any) continue;
        if (all) { acc += all_live; continue; }
        for (int u = u0; u < u1; ++u) {
          const int32_t* er = rows + (int64_t)u * rrec;
          for (int v = v0; v < v1; ++v) {
            const int32_t* ec = cols + (int64_t)v * crec;
            int L = 0;
            for (int p = 0; p < er[1]; ++p) {
              const uint8_t* Fr = F + (er[0] + p) * a.in.GW + ec[0];
              int lr = 0;
              for (int q = 0; q < ec[1]; ++q) lr += Fr[q] ? ec[3 + q] : 0;
              L += er[3 + p] * lr;
            }
            if (L > 0) acc += a.kk - er[2] * ec[2] + L;
          }
        }
      }
    }
    __shared__ long long red[4];
    acc = warp_sum_ll(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    contrib = red[0] + red[1] + red[2] + red[3];
  }
  const uint8_t nf = contrib > 0 || ((int64_t)cnt == total_in);
  const uint8_t of = a.out.fplane(s, 0)[t];
  for (int co = threadIdx.x; co < a.c_out; co += blockDim.x) a.out.fplane(s, co)[t] = nf;
  if (of && !nf) {  // tile went dead: restore the exact-zero invariant
    const int w = v1 - v0, n = (u1 - u0) * w;
    for (int e = threadIdx.x; e < n * a.c_out; e += blockDim.x) {
      const int co = e / n, l = e % n;
      a.out.plane(s, co)[(int64_t)(u0 + l / w) * h.Wo + v0 + l % w] = 0.0f;
    }
  }
  if (threadIdx.x == 0) {
    a.tile_active[(int64_t)s * T + t] = nf;
    if (contrib) atomicAdd(reinterpret_cast<unsigned long long*>(a.meter + s),
                           (unsigned long long)(2LL * a.c_out * contrib));
  }
}

// ---------------------------------------------------------------------------
// FFMA implicit GEMM over packed active sites
// ---------------------------------------------------------------------------
struct GemmArgs {
  TView in, out;
  const float* w;
  const float* bias;
  const int32_t* kdec;
  const int32_t* list;
  const int32_t* count;
  float* ws;
  int64_t mcap;  // capacity of packed sites (workspace row count)
  int c_in, c_out, kh, kw, stride, pad, K;
  int T, GWo, S;
  int splits, kchunk;
};

constexpr int BK = 8;

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) k_conv_gemm(GemmArgs a) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = (BN * BK + NT - 1) / NT;
  const int th = a.out.th, tw = a.out.tw, sites = th * tw;
  const int n_tiles = a.list ? *a.count : a.S * a.T;
  const int64_t M = (int64_t)n_tiles * sites;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  if (m0 >= M) return;
  const int n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int kbeg = z * a.kchunk, kend = min(a.K, kbeg + a.kchunk);

  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  __shared__ int64_t s_in[BM];   // session offset + y0*W + x0 into input, or -1
  __shared__ int64_t s_out[BM];  // session offset + u*Wo + v into output, or -1
  __shared__ int s_y0[BM], s_x0[BM];

  const int H = a.in.H, W = a.in.W, Ho = a.out.H, Wo = a.out.W;
  for (int m = threadIdx.x; m < BM; m += NT) {
    const int64_t pm = m0 + m;
    int64_t oi = -1, ii = 0;
    int y0 = -1000000, x0 = -1000000;
    if (pm < M) {
      const int e = (int)(pm / sites), l = (int)(pm % sites);
      const int ent = a.list ? a.list[e] : e;
      const int s = ent / a.T, t = ent % a.T;
      const int u = (t / a.GWo) * th + l / tw, v = (t % a.GWo) * tw + l % tw;
      if (u < Ho && v < Wo) {
        oi = (int64_t)s * a.out.vs + (int64_t)u * Wo + v;
        y0 = u * a.stride - a.pad;
        x0 = v * a.stride - a.pad;
        ii = (int64_t)s * a.in.vs + (int64_t)y0 * W + x0;
      }
    }
    s_in[m] = ii;
    s_out[m] = oi;
    s_y0[m] = y0;
    s_x0[m] = x0;
  }
  __syncthreads();

  const int tm = threadIdx.x % (BM / TM), tn = threadIdx.x / (BM / TM);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  float ra[A_PER], rb[B_PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      const int m = idx % BM, kk = idx / BM;
      const int k = k0 + kk;
      float v = 0.0f;
      if (k < kend) {
        const int off = __ldg(a.kdec + 2 * k), rq = __ldg(a.kdec + 2 * k + 1);
        const int iy = s_y0[m] + (rq >> 16), ix = s_x0[m] + (rq & 0xffff);
        if ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)W) v = __ldg(a.in.v + s_in[m] + off);
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      float v = 0.0f;
      if (idx < BN * BK) {
        const int n = idx / BK, kk = idx % BK;
        const int k = k0 + kk;
        if (k < kend && n0 + n < a.c_out) v = __ldg(a.w + (int64_t)(n0 + n) * a.K + k);
      }
      rb[e] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      As[buf][idx / BM][idx % BM] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      if (idx < BN * BK) Bs[buf][idx % BK][idx / BK] = rb[e];
    }
  };

  const int nk = (kend - kbeg + BK - 1) / BK;
  if (nk > 0) {
    load(kbeg);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
      const int cur = kt & 1;
      if (kt + 1 < nk) load(kbeg + (kt + 1) * BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(&As[cur][kk][tm * TM + i]);
          av[i] = t4.x; av[i + 1] = t4.y; av[i + 2] = t4.z; av[i + 3] = t4.w;
        }
        if constexpr (TN % 4 == 0) {
#pragma unroll
          for (int j = 0; j < TN; j += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tn * TN + j]);
            bv[j] = t4.x; bv[j + 1] = t4.y; bv[j + 2] = t4.z; bv[j + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < TN; ++j) bv[j] = Bs[cur][kk][tn * TN + j];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (kt + 1 < nk) store(cur ^ 1);
      __syncthreads();
    }
  }

  const int64_t plane = (int64_t)Ho * Wo;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = tm * TM + i;
    const int64_t pm = m0 + m;
    if (pm >= M) continue;
    const int64_t oi = s_out[m];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tn * TN + j;
      if (n >= a.c_out) continue;
      if (a.splits == 1) {
        if (oi >= 0) a.out.v[oi + n * plane] = a.bias ? __fadd_rn(acc[i][j], __ldg(a.bias + n)) : acc[i][j];
      } else {
        a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n] = acc[i][j];
      }
    }
  }
}

// deterministic split-K reduction + scatter
__global__ void k_conv_splitk_reduce(GemmArgs a) {
  const int th = a.out.th, tw = a.out.tw, sites = th * tw;
  const int n_tiles = a.list ? *a.count : a.S * a.T;
  const int64_t M = (int64_t)n_tiles * sites;
  const int Ho = a.out.H, Wo = a.out.W;
  const int64_t plane = (int64_t)Ho * Wo;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M * a.c_out;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pm = e / a.c_out;
    const int n = (int)(e % a.c_out);
    const int te = (int)(pm / sites), l = (int)(pm % sites);
    const int ent = a.list ? a.list[te] : te;
    const int s = ent / a.T, t = ent % a.T;
    const int u = (t / a.GWo) * th + l / tw, v = (t % a.GWo) * tw + l % tw;
    if (u >= Ho || v >= Wo) continue;
    float sum = 0.0f;
    for (int z = 0; z < a.splits; ++z) sum = __fadd_rn(sum, a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n]);
    if (a.bias) sum = __fadd_rn(sum, a.bias[n]);
    a.out.v[(int64_t)s * a.out.vs + n * plane + (int64_t)u * Wo + v] = sum;
  }
}

template <int BM, int BN, int TM, int TN>
static int launch_gemm(const GemmArgs& a, int64_t max_m, cudaStream_t st) {
  dim3 grid((unsigned)cdiv64(max_m, BM), (unsigned)cdiv(a.c_out, BN), (unsigned)a.splits);
  k_conv_gemm<BM, BN, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, st>>>(a);
  return 0;
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_conv_table_len(const evc_conv_geom* g) {
  if (!g) return -1;
  const int64_t K = (int64_t)g->c_in * g->kh * g->kw;
  return 8 + (int64_t)g->Ho * (3 + g->kh) + (int64_t)g->Wo * (3 + g->kw) + 2 * K;
}

int evc_conv_table_fill(const evc_conv_geom* g, int32_t* tab) {
  EVC_CHECK_ARG(g && tab, "conv_table_fill: null argument");
  EVC_CHECK_ARG(g->kh <= 0xffff && g->kw <= 0xffff && g->th > 0 && g->tw > 0, "conv_table_fill: geometry");
  const int K = g->c_in * g->kh * g->kw;
  TabHdr h;
  h.Ho = g->Ho;
  h.Wo = g->Wo;
  h.kh = g->kh;
  h.kw = g->kw;
  h.K = K;
  h.rows = 8;
  h.cols = h.rows + g->Ho * (3 + g->kh);
  h.kdec = h.cols + g->Wo * (3 + g->kw);
  memcpy(tab, &h, sizeof(h));
  axis_table(g->Ho, g->H, g->kh, g->stride, g->pad, g->th, tab + h.rows);
  axis_table(g->Wo, g->W, g->kw, g->stride, g->pad, g->tw, tab + h.cols);
  int32_t* kd = tab + h.kdec;
  for (int c = 0; c < g->c_in; ++c)
    for (int r = 0; r < g->kh; ++r)
      for (int q = 0; q < g->kw; ++q) {
        const int k = (c * g->kh + r) * g->kw + q;
        kd[2 * k] = c * g->H * g->W + r * g->W + q;
        kd[2 * k + 1] = (r << 16) | q;
      }
  return EVC_OK;
}

int evc_conv_mask(const evc_conv_geom* g, const evc_tensor* in, const evc_tensor* out, const int32_t* table,
                  const int32_t* in_true, uint8_t* tile_active, int64_t* meter, int32_t S, void* stream) {
  EVC_CHECK_ARG(g && in && out && table && in_true && tile_active && meter && S > 0, "conv_mask: null argument");
  EVC_CHECK_ARG(in->flags && out->flags, "conv_mask: masks required");
  MaskArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.tab = table;
  a.in_true = in_true;
  a.tile_active = tile_active;
  a.meter = meter;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kk = g->kh * g->kw;
  dim3 grid(a.out.GH * a.out.GW, S);
  k_conv_mask<<<grid, 128, 0, as_stream(stream)>>>(a);
  EVC_LAUNCH_CHECK("conv_mask");
  return EVC_OK;
}

int64_t evc_conv_workspace(const evc_conv_geom* g, int64_t max_tiles, int32_t splits) {
  if (!g || splits <= 1) return 0;
  return (int64_t)splits * max_tiles * g->th * g->tw * g->c_out;
}

int evc_conv_gemm(const evc_conv_geom* g, const evc_tensor* in, const float* weight, const float* bias,
                  const evc_tensor* out, const int32_t* table, const int32_t* tile_list, const int32_t* tile_count,
                  int32_t S, int32_t splits, float* workspace, void* stream) {
  EVC_CHECK_ARG(g && in && out && weight && table && S > 0 && splits >= 1, "conv_gemm: null argument");
  EVC_CHECK_ARG(!tile_list || tile_count, "conv_gemm: tile_count required with tile_list");
  EVC_CHECK_ARG(splits == 1 || workspace, "conv_gemm: workspace required for split-K");
  GemmArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.w = weight;
  a.bias = bias;
  TabHdr h;
  // the header lives on device; recompute host-side
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kh = g->kh;
  a.kw = g->kw;
  a.stride = g->stride;
  a.pad = g->pad;
  a.K = g->c_in * g->kh * g->kw;
  h.rows = 8;
  h.cols = h.rows + g->Ho * (3 + g->kh);
  h.kdec = h.cols + g->Wo * (3 + g->kw);
  a.kdec = table + h.kdec;
  a.list = tile_list;
  a.count = tile_count;
  a.T = a.out.GH * a.out.GW;
  a.GWo = a.out.GW;
  a.S = S;
  a.splits = splits;
  a.kchunk = (int)(cdiv64(cdiv64(a.K, splits), BK) * BK);
  a.ws = workspace;
  const int64_t max_m = (int64_t)S * a.T * g->th * g->tw;
  a.mcap = max_m;
  cudaStream_t st = as_stream(stream);
  if (g->c_out > 24 && g->c_out <= 32)
    launch_gemm<128, 32, 8, 4>(a, max_m, st);
  else if (g->c_out > 32)
    launch_gemm<128, 64, 8, 4>(a, max_m, st);
  else if (g->c_out > 4)
    launch_gemm<256, 16, 8, 4>(a, max_m, st);
  else
    launch_gemm<256, 4, 4, 2>(a, max_m, st);
  EVC_LAUNCH_CHECK("conv_gemm");
  if (splits > 1) {
    const int64_t work = max_m * g->c_out;
    const int blocks = (int)std::min<int64_t>(cdiv64(work, 256), 148 * 8);
    k_conv_splitk_reduce<<<blocks, 256, 0, st>>>(a);
    EVC_LAUNCH_CHECK("conv_splitk_reduce");
  }
  return EVC_OK;
}

}  // extern "C"

namespace evc {
int init_conv() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_conv_mask) != cudaSuccess) return EVC_ECUDA;
  return EVC_OK;
}
}  // namespace evc
