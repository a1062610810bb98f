// Mask propagation + exact FLOP meter of inc_conv2d (increment_ops.py:126-194).
//
// The reference meter (increment_ops.py:165-191) is
//   performed = 2*C_out * sum_c sum_{(u,v): L_c(u,v) > 0} (K^2 - inb(u,v) + L_c(u,v))
// with L_c the live in-bounds taps of site (u,v) in channel c and inb its
// in-bounds taps.  Split it:
//   sum_{sites} L_c = sum_{a,b} F_c[a][b] * RT[a] * CT[b]          (all sites,
//        because L_c = 0 contributes nothing; RT/CT are static tap counts per
//        input tile row/column), and
//   sum_{sites with L_c>0} (K^2 - inb)                              (nonzero
//        only at output sites whose taps hit the zero padding: the border).
// So one pass over the input flags gives the bulk of the meter as a weighted
// count (k_conv_count) and only border sites need a per-site check
// (k_conv_flags).  Output tiles: live iff any channel has a live input tile in
// the tile's receptive box, broadcast over C_out.  The
// all-false / all-true shortcuts (increment_ops.py:148-154) are applied from
// the exact live-flag count.

#include "conv_common.cuh"

namespace evc {

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

static void axis_sums(const int32_t* axis, int n_out, int k, int32_t* tot) {
  for (int u = 0; u < n_out; ++u) {
    const int32_t* e = axis + (int64_t)u * (3 + k);
    for (int q = 0; q < e[1]; ++q) tot[e[0] + q] += e[3 + q];
  }
}

static void axis_boxes(const int32_t* axis, int n_out, int k, int tile, int32_t* box) {
  const int ntile = (n_out + tile - 1) / tile;
  for (int i = 0; i < ntile; ++i) {
    int lo = 1 << 30, hi = -1, border = 0;
    for (int u = i * tile; u < std::min(n_out, (i + 1) * tile); ++u) {
      const int32_t* e = axis + (int64_t)u * (3 + k);
      if (e[1]) {
        lo = std::min(lo, e[0]);
        hi = std::max(hi, e[0] + e[1] - 1);
      }
      border |= (e[2] > 0 && e[2] < k);
    }
    box[3 * i] = hi < 0 ? 0 : lo;
    box[3 * i + 1] = hi;
    box[3 * i + 2] = border;
  }
}

struct MaskArgs {
  TView in, out;
  const int32_t* tab;
  int32_t* fany;    // [S][GHi*GWi]   OR over channels of the input flags
  int64_t* term1;   // [S]            sum_c sum_ab F*RT*CT
  int32_t* in_true;  // [S]            live input flags
  int32_t* list;
  int32_t* count;
  int64_t* meter;
  int64_t dense;    // 2*K^2*C_in*C_out*Ho*Wo
  int c_in, c_out, kk;
};

constexpr int kCountCh = 32;

// One thread per input tile, kCountCh channels per block row.
__global__ void __launch_bounds__(128) k_conv_count(MaskArgs a) {
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int Ti = h.GHi * h.GWi;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.z;
  const int c0 = blockIdx.y * kCountCh, c1 = min(a.c_in, c0 + kCountCh);
  int cnt = 0;
  long long wsum = 0;
  if (t < Ti) {
    const uint8_t* f = a.in.f + (int64_t)s * a.in.fs + t;
    for (int c = c0; c < c1; ++c) cnt += f[(int64_t)c * Ti] != 0;
    if (cnt) {
      a.fany[(int64_t)s * Ti + t] = 1;  // benign race: every writer stores 1
      wsum = (long long)cnt * a.tab[h.rt + t / h.GWi] * a.tab[h.ct + t % h.GWi];
    }
  }
  __shared__ int s_c[4];
  __shared__ long long s_w[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  }
  if (lane == 0) {
    s_c[wid] = cnt;
    s_w[wid] = wsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int c = s_c[0] + s_c[1] + s_c[2] + s_c[3];
    const long long w = s_w[0] + s_w[1] + s_w[2] + s_w[3];
    if (c) atomicAdd(a.in_true + s, c);
    if (w) atomicAdd(reinterpret_cast<unsigned long long*>(a.term1 + s), (unsigned long long)w);
  }
}

// One CTA per (output tile, session).
__global__ void __launch_bounds__(64) k_conv_flags(MaskArgs a) {
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int t = blockIdx.x, s = blockIdx.y;
  const int To = h.GHo * h.GWo, Ti = h.GHi * h.GWi;
  const int i = t / h.GWo, j = t % h.GWo;
  const int th = a.out.th, tw = a.out.tw;
  const int u0 = i * th, u1 = min(h.Ho, u0 + th);
  const int v0 = j * tw, v1 = min(h.Wo, v0 + tw);
  const int* br = a.tab + h.boxr + 3 * i;
  const int* bc = a.tab + h.boxc + 3 * j;
  const int cnt = a.in_true[s];
  const bool all_false = cnt == 0;
  const bool all_true = (int64_t)cnt == (int64_t)a.c_in * Ti;
  bool nf = all_true;
  if (!all_true && !all_false && br[1] >= br[0] && bc[1] >= bc[0]) {
    const int32_t* fa = a.fany + (int64_t)s * Ti;
    int any = 0;
    for (int e = threadIdx.x; e < (br[1] - br[0] + 1) * (bc[1] - bc[0] + 1); e += blockDim.x) {
      const int w = bc[1] - bc[0] + 1;
      any |= fa[(br[0] + e / w) * h.GWi + bc[0] + e % w];
    }
    nf = __syncthreads_or(any) != 0;
  }
  // padding-tap correction at border sites (sum over live channels of K^2 - inb)
  if (nf && !all_true && (br[2] || bc[2])) {
    long long acc = 0;
    const int32_t* rows = a.tab + h.rows;
    const int32_t* cols = a.tab + h.cols;
    for (int u = u0; u < u1; ++u) {
      const int32_t* er = rows + (int64_t)u * (3 + h.kh);
      if (!er[1]) continue;
      for (int v = v0; v < v1; ++v) {
        const int32_t* ec = cols + (int64_t)v * (3 + h.kw);
        const int D = a.kk - er[2] * ec[2];
        if (!ec[1] || D == 0) continue;
        for (int c = threadIdx.x; c < a.c_in; c += blockDim.x) {
          const uint8_t* F = a.in.fplane(s, c);
          int live = 0;
          for (int p = 0; p < er[1]; ++p)
            for (int q = 0; q < ec[1]; ++q) live |= F[(er[0] + p) * a.in.GW + ec[0] + q];
          acc += live ? D : 0;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ long long s_a[2];
    if ((threadIdx.x & 31) == 0) s_a[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0 && s_a[0] + s_a[1])
      atomicAdd(reinterpret_cast<unsigned long long*>(a.meter + s),
                (unsigned long long)(2LL * a.c_out * (s_a[0] + s_a[1])));
  }
  if (t == 0 && threadIdx.x == 0) {
    const long long base = all_true ? a.dense : (all_false ? 0 : 2LL * a.c_out * a.term1[s]);
    if (base) atomicAdd(reinterpret_cast<unsigned long long*>(a.meter + s), (unsigned long long)base);
  }
  const uint8_t of = a.out.fplane(s, 0)[t];
  for (int co = threadIdx.x; co < a.c_out; co += blockDim.x) a.out.fplane(s, co)[t] = nf;
  if (of && !nf) {  // tile went dead: restore the exact-zero invariant
    const int w = v1 - v0, n = (u1 - u0) * w;
    for (int e = threadIdx.x; e < n * a.c_out; e += blockDim.x) {
      const int co = e / n, l = e % n;
      a.out.plane(s, co)[(int64_t)(u0 + l / w) * h.Wo + v0 + l % w] = 0.0f;
    }
  }
  if (nf && threadIdx.x == 0) a.list[atomicAdd(a.count, 1)] = s * To + t;
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_conv_table_len(const evc_conv_geom* g) { return g ? tab_len(g) : -1; }

int evc_conv_table_fill(const evc_conv_geom* g, int32_t* tab) {
  EVC_CHECK_ARG(g && tab, "conv_table_fill: null argument");
  EVC_CHECK_ARG(g->kh <= 0xffff && g->kw <= 0xffff && g->th > 0 && g->tw > 0, "conv_table_fill: geometry");
  const TabHdr h = tab_layout(g);
  memset(tab, 0, sizeof(int32_t) * (size_t)tab_len(g));
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
  axis_sums(tab + h.rows, g->Ho, g->kh, tab + h.rt);
  axis_sums(tab + h.cols, g->Wo, g->kw, tab + h.ct);
  axis_boxes(tab + h.rows, g->Ho, g->kh, g->th, tab + h.boxr);
  axis_boxes(tab + h.cols, g->Wo, g->kw, g->tw, tab + h.boxc);
  return EVC_OK;
}

int64_t evc_conv_mask_scratch(const evc_conv_geom* g, int32_t S) {
  if (!g) return -1;
  const TabHdr h = tab_layout(g);
  return ((int64_t)S * h.GHi * h.GWi + 1) / 2 * 2 + 2LL * S;
}

int evc_conv_mask(const evc_conv_geom* g, const evc_tensor* in, const evc_tensor* out, const int32_t* table,
                  int32_t* scratch, int32_t* in_true, int32_t* tile_list, int32_t* tile_count, int64_t* meter,
                  int32_t S, void* stream) {
  EVC_CHECK_ARG(g && in && out && table && scratch && in_true && tile_list && tile_count && meter && S > 0,
                "conv_mask: null argument");
  EVC_CHECK_ARG(in->flags && out->flags, "conv_mask: masks required");
  const TabHdr h = tab_layout(g);
  MaskArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.tab = table;
  a.fany = scratch;
  a.term1 = reinterpret_cast<int64_t*>(scratch + ((int64_t)S * h.GHi * h.GWi + 1) / 2 * 2);
  a.in_true = in_true;
  a.list = tile_list;
  a.count = tile_count;
  a.meter = meter;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kk = g->kh * g->kw;
  a.dense = 2LL * a.kk * g->c_in * g->c_out * g->Ho * g->Wo;
  cudaStream_t st = as_stream(stream);
  dim3 g1(cdiv(h.GHi * h.GWi, 128), cdiv(g->c_in, kCountCh), S);
  k_conv_count<<<g1, 128, 0, st>>>(a);
  EVC_LAUNCH_CHECK("conv_count");
  k_conv_flags<<<dim3(h.GHo * h.GWo, S), 64, 0, st>>>(a);
  EVC_LAUNCH_CHECK("conv_flags");
  return EVC_OK;
}

}  // extern "C"

namespace evc {
int init_conv_mask() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_conv_flags) != cudaSuccess) return EVC_ECUDA;
  return EVC_OK;
}
}  // namespace evc
