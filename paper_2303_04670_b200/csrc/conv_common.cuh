// Static per-conv-layer table shared by the mask/meter and GEMM kernels.
#pragma once

#include "common.cuh"

namespace evc {

// int32 table layout (all offsets in int32 entries from the table start):
//   [0..15] header (TabHdr)
//   rows  : Ho  x (3 + kh)  a_first, n_a, inR, cnt[kh]   (input tile rows hit by output row u)
//   cols  : Wo  x (3 + kw)  b_first, n_b, inC, cnt[kw]
//   kdec  : K   x 2         c*H*W + r*W + q,  (r << 16) | q      (k = (c*kh + r)*kw + q)
//   rt    : GHi             RT[a] = sum_u cnt(u, a)   (output-row/tap pairs landing in input tile row a)
//   ct    : GWi             CT[b]
//   boxr  : GHo x 3         A0, A1, has_border_row   (input tile-row box of output tile row i)
//   boxc  : GWo x 3         B0, B1, has_border_col
struct TabHdr {
  int Ho, Wo, kh, kw, K, GHi, GWi, GHo, GWo;
  int rows, cols, kdec, rt, ct, boxr, boxc;
};

static inline TabHdr tab_layout(const evc_conv_geom* g) {
  TabHdr h;
  h.Ho = g->Ho;
  h.Wo = g->Wo;
  h.kh = g->kh;
  h.kw = g->kw;
  h.K = g->c_in * g->kh * g->kw;
  h.GHi = (g->H + g->th - 1) / g->th;
  h.GWi = (g->W + g->tw - 1) / g->tw;
  h.GHo = (g->Ho + g->th - 1) / g->th;
  h.GWo = (g->Wo + g->tw - 1) / g->tw;
  h.rows = 16;
  h.cols = h.rows + g->Ho * (3 + g->kh);
  h.kdec = h.cols + g->Wo * (3 + g->kw);
  h.rt = h.kdec + 2 * h.K;
  h.ct = h.rt + h.GHi;
  h.boxr = h.ct + h.GWi;
  h.boxc = h.boxr + 3 * h.GHo;
  return h;
}

static inline int64_t tab_len(const evc_conv_geom* g) {
  const TabHdr h = tab_layout(g);
  return h.boxc + 3 * h.GWo;
}

}  // namespace evc
