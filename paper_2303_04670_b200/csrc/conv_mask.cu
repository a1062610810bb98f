// Mask propagation + exact FLOP meter of inc_conv2d (increment_ops.py:126-194).
//
// The reference meter (increment_ops.py:165-191) is
//   performed = 2*C_out * sum_c sum_{(u,v): L_c(u,v) > 0} (K^2 - inb(u,v) + L_c(u,v))
// with L_c the live in-bounds taps of site (u,v) in channel c and inb its
// in-bounds taps.  It splits into
//   sum_{all sites} L_c = sum_{a,b} F_c[a][b] * RT[a] * CT[b]
// (sites with L_c = 0 add nothing; RT/CT are static tap counts per input tile
// row / column), plus
//   sum_{sites with L_c > 0} (K^2 - inb)
// which is nonzero only at border sites whose taps hit the zero padding; the
// host groups those sites by their input-tile box, so the device work is one
// OR over <= a few flags per (group, channel).  Both terms are computed fully
// in parallel by k_conv_count; k_conv_flags then decides each output tile
// (live iff some input tile in its receptive box is live in any channel,
// SURVEY.md A.1) and applies the all-false / all-true shortcuts
// (increment_ops.py:148-154) from the exact live-flag count.

#include <map>
#include <tuple>
#include <vector>

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
    int lo = 1 << 30, hi = -1;
    for (int u = i * tile; u < std::min(n_out, (i + 1) * tile); ++u) {
      const int32_t* e = axis + (int64_t)u * (3 + k);
      if (e[1]) {
        lo = std::min(lo, e[0]);
        hi = std::max(hi, e[0] + e[1] - 1);
      }
    }
    box[2 * i] = hi < 0 ? 0 : lo;
    box[2 * i + 1] = hi;
  }
}

// border sites grouped by input-tile box -> (a0, na, b0, nb, sumD)
static std::vector<int32_t> border_groups(const evc_conv_geom* g, const int32_t* rows, const int32_t* cols) {
  std::map<std::tuple<int, int, int, int>, int64_t> m;
  const int kk = g->kh * g->kw;
  for (int u = 0; u < g->Ho; ++u) {
    const int32_t* er = rows + (int64_t)u * (3 + g->kh);
    if (!er[1]) continue;
    for (int v = 0; v < g->Wo; ++v) {
      const int32_t* ec = cols + (int64_t)v * (3 + g->kw);
      const int D = kk - er[2] * ec[2];
      if (!ec[1] || D == 0) continue;
      m[std::make_tuple(er[0], er[1], ec[0], ec[1])] += D;
    }
  }
  std::vector<int32_t> out;
  for (auto& kv : m) {
    out.push_back(std::get<0>(kv.first));
    out.push_back(std::get<1>(kv.first));
    out.push_back(std::get<2>(kv.first));
    out.push_back(std::get<3>(kv.first));
    out.push_back((int32_t)kv.second);
  }
  return out;
}

// Full table; returns its length (entries) and fills `tab` when non-null.
static int64_t build_table(const evc_conv_geom* g, int32_t* tab) {
  TabHdr h = tab_layout(g);
  std::vector<int32_t> rows((size_t)g->Ho * (3 + g->kh)), cols((size_t)g->Wo * (3 + g->kw));
  axis_table(g->Ho, g->H, g->kh, g->stride, g->pad, g->th, rows.data());
  axis_table(g->Wo, g->W, g->kw, g->stride, g->pad, g->tw, cols.data());
  const std::vector<int32_t> grp = border_groups(g, rows.data(), cols.data());
  h.ngrp = (int)(grp.size() / 5);
  const int64_t len = h.grp + (int64_t)grp.size();
  if (!tab) return len;
  memset(tab, 0, sizeof(int32_t) * (size_t)len);
  memcpy(tab, &h, sizeof(h));
  memcpy(tab + h.rows, rows.data(), rows.size() * sizeof(int32_t));
  memcpy(tab + h.cols, cols.data(), cols.size() * sizeof(int32_t));
  int32_t* kd = tab + h.kdec;
  for (int c = 0; c < g->c_in; ++c)
    for (int r = 0; r < g->kh; ++r)
      for (int q = 0; q < g->kw; ++q) {
        const int k = (c * g->kh + r) * g->kw + q;
        kd[2 * k] = c * g->H * g->W + r * g->W + q;
        kd[2 * k + 1] = (r << 16) | q;
      }
  axis_sums(rows.data(), g->Ho, g->kh, tab + h.rt);
  axis_sums(cols.data(), g->Wo, g->kw, tab + h.ct);
  axis_boxes(rows.data(), g->Ho, g->kh, g->th, tab + h.boxr);
  axis_boxes(cols.data(), g->Wo, g->kw, g->tw, tab + h.boxc);
  if (!grp.empty()) memcpy(tab + h.grp, grp.data(), grp.size() * sizeof(int32_t));
  return len;
}

struct MaskArgs {
  TView in, out;
  const int32_t* tab;
  int32_t* fany;     // [S][GHi*GWi]   1 where any channel's input tile is live
  int64_t* bulk;     // [S]            sum_c sum_ab F*RT*CT + border padding term
  int32_t* in_true;  // [S]            live input flags
  int32_t* list;
  int32_t* count;
  uint8_t* regions;  // optional [S][RHn*RWn] flags of 4x32 output regions (TMA GEMM work)
  int64_t* meter;
  int64_t dense;  // 2*K^2*C_in*C_out*Ho*Wo
  int c_in, c_out, nb_count, RHn, RWn;
};

constexpr int kCountThreads = 256;

__global__ void __launch_bounds__(kCountThreads) k_conv_count(MaskArgs a) {
  pdl_wait();
  pdl_trigger();
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int Ti = h.GHi * h.GWi;
  const int s = blockIdx.y;
  int cnt = 0;
  long long w = 0;
  if ((int)blockIdx.x < a.nb_count) {  // weighted live-flag count over (channel, tile)
    const int64_t e = (int64_t)blockIdx.x * kCountThreads + threadIdx.x;
    if (e < (int64_t)a.c_in * Ti) {
      const int t = (int)(e % Ti);
      if (a.in.f[(int64_t)s * a.in.fs + e]) {
        a.fany[(int64_t)s * Ti + t] = 1;  // benign race: every writer stores 1
        cnt = 1;
        w = (long long)a.tab[h.rt + t / h.GWi] * a.tab[h.ct + t % h.GWi];
      }
    }
  } else {  // border padding term over (group, channel)
    const int64_t e = (int64_t)(blockIdx.x - a.nb_count) * kCountThreads + threadIdx.x;
    if (e < (int64_t)h.ngrp * a.c_in) {
      const int g = (int)(e / a.c_in), c = (int)(e % a.c_in);
      const int32_t* gp = a.tab + h.grp + 5 * g;
      const uint8_t* F = a.in.fplane(s, c);
      int live = 0;
      for (int p = 0; p < gp[1]; ++p)
        for (int q = 0; q < gp[3]; ++q) live |= F[(gp[0] + p) * h.GWi + gp[2] + q];
      if (live) w = gp[4];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  __shared__ int s_c[kCountThreads / 32];
  __shared__ long long s_w[kCountThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_c[wid] = cnt;
    s_w[wid] = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    long long ww = 0;
    for (int q = 0; q < kCountThreads / 32; ++q) {
      c += s_c[q];
      ww += s_w[q];
    }
    if (c) atomicAdd(a.in_true + s, c);
    if (ww) atomicAdd(reinterpret_cast<unsigned long long*>(a.bulk + s), (unsigned long long)ww);
  }
}

// One warp per (output tile, session).
__global__ void __launch_bounds__(256) k_conv_flags(MaskArgs a) {
  pdl_wait();
  pdl_trigger();
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int To = h.GHo * h.GWo, Ti = h.GHi * h.GWi;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int s = blockIdx.y;
  const int cnt = a.in_true[s];
  const bool all_false = cnt == 0;
  const bool all_true = (int64_t)cnt == (int64_t)a.c_in * Ti;
  if (t == 0 && lane == 0) {
    const long long base = all_true ? a.dense : (all_false ? 0 : 2LL * a.c_out * a.bulk[s]);
    if (base) atomicAdd(reinterpret_cast<unsigned long long*>(a.meter + s), (unsigned long long)base);
  }
  if (t >= To) return;
  const int i = t / h.GWo, j = t % h.GWo;
  const int* br = a.tab + h.boxr + 2 * i;
  const int* bc = a.tab + h.boxc + 2 * j;
  bool nf = all_true;
  if (!all_true && !all_false && br[1] >= br[0] && bc[1] >= bc[0]) {
    const int32_t* fa = a.fany + (int64_t)s * Ti;
    const int w = bc[1] - bc[0] + 1;
    int any = 0;
    for (int e = lane; e < (br[1] - br[0] + 1) * w; e += 32) any |= fa[(br[0] + e / w) * h.GWi + bc[0] + e % w];
    nf = __any_sync(0xffffffffu, any) != 0;
  }
  const uint8_t of = a.out.fplane(s, 0)[t];
  __syncwarp();
  for (int co = lane; co < a.c_out; co += 32) a.out.fplane(s, co)[t] = nf;
  if (of && !nf) {  // tile went dead: restore the exact-zero invariant
    const int th = a.out.th, tw = a.out.tw;
    const int u0 = i * th, u1 = min(h.Ho, u0 + th), v0 = j * tw, v1 = min(h.Wo, v0 + tw);
    const int wd = v1 - v0, n = (u1 - u0) * wd;
    for (int e = lane; e < n * a.c_out; e += 32) {
      const int co = e / n, l = e % n;
      a.out.plane(s, co)[(int64_t)(u0 + l / wd) * h.Wo + v0 + l % wd] = 0.0f;
    }
  }
  if (nf && lane == 0) {
    if (a.list) a.list[atomicAdd(a.count, 1)] = s * To + t;
    if (a.regions) {  // mark the 4x32 output regions this tile overlaps (benign races: all store 1)
      const int th = a.out.th, tw = a.out.tw;
      const int ulast = min(h.Ho, (i + 1) * th) - 1, vlast = min(h.Wo, (j + 1) * tw) - 1;
      for (int ri = (i * th) / 4; ri <= ulast / 4; ++ri)
        for (int rj = (j * tw) / 32; rj <= vlast / 32; ++rj)
          a.regions[((int64_t)s * a.RHn + ri) * a.RWn + rj] = 1;
    }
  }
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_conv_table_len(const evc_conv_geom* g) { return g ? build_table(g, nullptr) : -1; }

int evc_conv_table_fill(const evc_conv_geom* g, int32_t* tab) {
  EVC_CHECK_ARG(g && tab, "conv_table_fill: null argument");
  EVC_CHECK_ARG(g->kh <= 0xffff && g->kw <= 0xffff && g->th > 0 && g->tw > 0, "conv_table_fill: geometry");
  build_table(g, tab);
  return EVC_OK;
}

int64_t evc_conv_mask_scratch(const evc_conv_geom* g, int32_t S) {
  if (!g) return -1;
  const TabHdr h = tab_layout(g);
  return ((int64_t)S * h.GHi * h.GWi + 1) / 2 * 2 + 2LL * S;
}

int evc_conv_mask(const evc_conv_geom* g, const evc_tensor* in, const evc_tensor* out, const int32_t* table,
                  int32_t* scratch, int32_t* in_true, int32_t* tile_list, int32_t* tile_count,
                  uint8_t* region_flags, int64_t* meter, int32_t S, void* stream) {
  EVC_CHECK_ARG(g && in && out && table && scratch && in_true && meter && S > 0, "conv_mask: null argument");
  EVC_CHECK_ARG((tile_list != nullptr) == (tile_count != nullptr), "conv_mask: tile_list needs tile_count");
  EVC_CHECK_ARG(in->flags && out->flags, "conv_mask: masks required");
  const TabHdr h = tab_layout(g);
  // number of border groups is static per geometry; recompute it host-side
  static thread_local std::map<std::tuple<int, int, int, int, int, int, int, int, int, int>, int> ngrp_cache;
  const auto key = std::make_tuple(g->c_in, g->kh, g->kw, g->stride, g->pad, g->H, g->W, g->th, g->tw, g->Ho);
  auto it = ngrp_cache.find(key);
  int ngrp;
  if (it == ngrp_cache.end()) {
    const int64_t len = build_table(g, nullptr);
    ngrp = (int)((len - h.grp) / 5);
    ngrp_cache[key] = ngrp;
  } else {
    ngrp = it->second;
  }
  MaskArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.tab = table;
  a.fany = scratch;
  a.bulk = reinterpret_cast<int64_t*>(scratch + ((int64_t)S * h.GHi * h.GWi + 1) / 2 * 2);
  a.in_true = in_true;
  a.list = tile_list;
  a.count = tile_count;
  a.regions = region_flags;
  a.RHn = (g->Ho + 3) / 4;
  a.RWn = (g->Wo + 31) / 32;
  a.meter = meter;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.dense = 2LL * g->kh * g->kw * g->c_in * g->c_out * g->Ho * g->Wo;
  a.nb_count = (int)cdiv64((int64_t)g->c_in * h.GHi * h.GWi, kCountThreads);
  const int nb_border = (int)cdiv64((int64_t)ngrp * g->c_in, kCountThreads);
  cudaStream_t st = as_stream(stream);
  launch_pdl(k_conv_count, dim3(dim3(a.nb_count + nb_border, S)), dim3(kCountThreads), 0, st, a);
  EVC_LAUNCH_CHECK("conv_count");
  launch_pdl(k_conv_flags, dim3(dim3(cdiv(h.GHo * h.GWo, 8), S)), dim3(256), 0, st, a);
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
