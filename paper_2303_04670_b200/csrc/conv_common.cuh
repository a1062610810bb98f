// Static per-conv-layer table shared by the mask/meter and GEMM kernels.
#pragma once

#include "common.cuh"

namespace evc {

// int32 table layout (all offsets in int32 entries from the table start):
//   [0..19] header (TabHdr)
//   rows  : Ho  x (3 + kh)  a_first, n_a, inR, cnt[kh]   (input tile rows hit by output row u)
//   cols  : Wo  x (3 + kw)  b_first, n_b, inC, cnt[kw]
//   kdec  : K   x 2         c*H*W + r*W + q,  (r << 16) | q      (k = (c*kh + r)*kw + q)
//   rt    : GHi             RT[a] = sum_u cnt(u, a)   (output-row/tap pairs landing in input tile row a)
//   ct    : GWi             CT[b]
//   boxr  : GHo x 2         A0, A1   (input tile-row box of output tile row i; A1 < A0 if empty)
//   boxc  : GWo x 2         B0, B1
//   grp   : ngrp x 5        a0, na, b0, nb, sumD: border output sites with the same
//                           input tile box, sumD = sum over them of (K^2 - inb) > 0
struct TabHdr {
  int Ho, Wo, kh, kw, K, GHi, GWi, GHo, GWo;
  int rows, cols, kdec, rt, ct, boxr, boxc, grp, ngrp, pad0, pad1;
};

// Header with every offset except the border groups (grp, ngrp filled by the host builder).
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
  h.rows = 20;
  h.cols = h.rows + g->Ho * (3 + g->kh);
  h.kdec = h.cols + g->Wo * (3 + g->kw);
  h.rt = h.kdec + 2 * h.K;
  h.ct = h.rt + h.GHi;
  h.boxr = h.ct + h.GWi;
  h.boxc = h.boxr + 2 * h.GHo;
  h.grp = h.boxc + 2 * h.GWo;
  h.ngrp = 0;
  h.pad0 = h.pad1 = 0;
  return h;
}

// tcgen05 path (conv_tc.cu): launches the tensor-core GEMM; returns the
// effective number of K-splits (>= 1) or a negative EVC_E* code.
int conv_tc_launch(const evc_conv_geom* g, const evc_tensor* in, const float* wpack, const float* bias,
                   const evc_tensor* out, const int32_t* table, const int32_t* tile_list, const int32_t* tile_count,
                   int32_t S, int32_t splits, float* workspace, cudaStream_t st);
int init_conv_tc();

}  // namespace evc
