// inc_linear (increment_ops.py:197-223) and event binning (events.py:251-292).

#include <cub/cub.cuh>

#include "common.cuh"

namespace evc {

// ---------------------------------------------------------------------------
// inc_linear + flatten_increment: runs of th*tw flat elements whose liveness
// is recomputed from values (make_tile_mask on the (1,1,L) view,
// increment_ops.py:197-202).  One CTA owns a chunk of whole runs, stages the
// live values in shared memory, and writes per-row partial dot products;
// a second kernel reduces the chunks in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kLinChunk = 2048;

// chunk = whole number of runs, close to kLinChunk
static inline int lin_chunk(int run) {
  const int c = (kLinChunk / run) * run;
  return c > 0 ? c : run;
}

__global__ void __launch_bounds__(256) k_linear_partial(const float* __restrict__ x, int64_t xs, int64_t L, int run,
                                                        int chunk, const float* __restrict__ Wt, int F, int dense,
                                                        const uint8_t* __restrict__ runflags, int64_t rfs,
                                                        float* __restrict__ part, int64_t* meter) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_x[];
  __shared__ int s_live_elems;
  const int b = blockIdx.x, s = blockIdx.y;
  const int64_t c0 = (int64_t)b * chunk;
  const int n = (int)(L - c0 < chunk ? L - c0 : chunk);
  const float* xv = x + (int64_t)s * xs + c0;
  if (threadIdx.x == 0) s_live_elems = 0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s_x[e] = xv[e];
  __syncthreads();
  // run liveness (warp per run)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nruns = (n + run - 1) / run;
  for (int r = wid; r < nruns; r += nw) {
    const int r0 = r * run, r1 = min(n, r0 + run);
    bool nz = false;
    if (runflags) {  // caller-supplied (1,1,L) mask with tile (1, run)
      nz = runflags[(int64_t)s * rfs + c0 / run + r] != 0;
    } else {
      for (int e = r0 + lane; e < r1; e += 32) nz |= s_x[e] != 0.0f;
      nz = __any_sync(0xffffffffu, nz);
    }
    nz = nz || dense;
    if (!nz)
      for (int e = r0 + lane; e < r1; e += 32) s_x[e] = 0.0f;  // already zero; keeps -0.0 out
    else if (lane == 0)
      atomicAdd(&s_live_elems, r1 - r0);
  }
  __syncthreads();
  if (!dense && threadIdx.x == 0 && s_live_elems)
    atomicAdd(reinterpret_cast<unsigned long long*>(meter + s), (unsigned long long)(2LL * F * s_live_elems));
  if (!dense && s_live_elems == 0) {
    for (int f = threadIdx.x; f < F; f += blockDim.x) part[((int64_t)s * gridDim.x + b) * F + f] = 0.0f;
    return;
  }
  for (int f = wid; f < F; f += nw) {
    const float* wr = Wt + (int64_t)f * L + c0;
    float acc = 0.0f;
    for (int e = lane; e < n; e += 32) {
      const float v = s_x[e];
      if (v != 0.0f) acc = fmaf(__ldg(wr + e), v, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) part[((int64_t)s * gridDim.x + b) * F + f] = acc;
  }
}

__global__ void k_linear_reduce(const float* __restrict__ part, int nchunks, int F, const float* __restrict__ bias,
                                float* __restrict__ y, int64_t ys, uint8_t* flags, int64_t fs) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int b = 0; b < nchunks; ++b) acc = __fadd_rn(acc, part[((int64_t)s * nchunks + b) * F + f]);
    if (bias) acc = __fadd_rn(acc, bias[f]);
    y[(int64_t)s * ys + f] = acc;
    if (flags) flags[(int64_t)s * fs + f] = 1;  // output mask all-true (increment_ops.py:223)
  }
}

// ---------------------------------------------------------------------------
// encode: stable radix sort of the window by pixel key, then one thread per
// key run folds its events in time order -> no atomics, bit-exact.
// ---------------------------------------------------------------------------
__global__ void k_event_keys(const uint16_t* __restrict__ x, const uint16_t* __restrict__ y,
                             const int8_t* __restrict__ p, int64_t lo, int n, int H, int W, int kind,
                             uint32_t* keys, int32_t* vals) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t e = lo + i;
  uint32_t k = (uint32_t)y[e] * (uint32_t)W + x[e];
  if (kind != EVC_ENC_VOXEL && p[e] <= 0) k += (uint32_t)(H * W);
  keys[i] = k;
  vals[i] = (int32_t)e;
}

__global__ void k_event_runs(const uint64_t* __restrict__ t, const int8_t* __restrict__ p,
                             const uint32_t* __restrict__ keys, const int32_t* __restrict__ ev, int n, int64_t t0,
                             int64_t delta, int HW, int kind, int bins, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;  // not a run head
  int j = i + 1;
  while (j < n && keys[j] == key) ++j;
  const double dt0 = (double)t0, dd = (double)delta;
  if (kind == EVC_ENC_COUNT) {
    out[key] = (float)(j - i);  // integer counts, exact (events.py:267-272)
    return;
  }
  if (kind == EVC_ENC_TIMESTAMP) {
    float m = 0.0f;  // np.maximum.at over zeros (events.py:274-280)
    for (int q = i; q < j; ++q) {
      const double rel = ((double)t[ev[q]] - dt0) / dd;
      m = fmaxf(m, __double2float_rn(rel));
    }
    out[key] = m;
    return;
  }
  // voxel (events.py:282-292): pass 1 adds p*(1-frac) to bin lo for every
  // event in time order, pass 2 adds p*frac to bin lo+1; each add rounds
  // f32(f64(acc) + v) like np.add.at on a float32 array.
  float acc[32];
  for (int b = 0; b < bins; ++b) acc[b] = 0.0f;
  for (int pass = 0; pass < 2; ++pass) {
    for (int q = i; q < j; ++q) {
      const int e = ev[q];
      const double rel = ((double)t[e] - dt0) / dd;
      const float ts = __double2float_rn(rel * (double)(bins - 1));
      const long long b0 = (long long)floorf(ts);
      const double frac = (double)ts - (double)b0;
      const double pv = (double)(float)p[e];
      const long long b = pass ? b0 + 1 : b0;
      const double v = pass ? pv * frac : pv * (1.0 - frac);
      if (b >= 0 && b < bins) acc[b] = __double2float_rn((double)acc[b] + v);
    }
  }
  for (int b = 0; b < bins; ++b) out[(int64_t)b * HW + key] = acc[b];
}

static int bits_for(uint32_t maxkey) {
  int b = 1;
  while (b < 32 && (1ull << b) <= maxkey) ++b;
  return b;
}

static size_t cub_temp_bytes(int64_t n, int end_bit) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs<uint32_t, int32_t>(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                     (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0, end_bit);
  return bytes;
}

static inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_linear_workspace(int32_t F, int64_t L, int32_t run, int32_t S) {
  return (int64_t)S * cdiv64(L, lin_chunk(run > 0 ? run : 1)) * F;
}

int evc_linear(const evc_tensor* in, const float* weight, const float* bias, const evc_tensor* out, int32_t F,
               int32_t dense, int64_t* meter, float* workspace, int32_t S, void* stream) {
  EVC_CHECK_ARG(in && out && weight && workspace && S > 0 && F > 0, "linear: null argument");
  EVC_CHECK_ARG(dense || meter, "linear: meter required");
  const int64_t L = (int64_t)in->C * in->H * in->W;
  const int run = in->th * in->tw;
  EVC_CHECK_ARG(!in->flags || (in->C == 1 && in->H == 1 && in->th == 1), "linear: masked input must be (1,1,L)");
  const int chunk = lin_chunk(run);
  const int nchunks = (int)cdiv64(L, chunk);
  cudaStream_t st = as_stream(stream);
  launch_pdl(k_linear_partial, dim3(dim3(nchunks, S)), dim3(256), chunk * sizeof(float), st, in->vals, in->vstride, L, run, chunk,
                                                                         weight, F, dense, in->flags, in->fstride,
                                                                         workspace, meter);
  EVC_LAUNCH_CHECK("linear_partial");
  launch_pdl(k_linear_reduce, dim3(dim3(cdiv(F, 128), S)), dim3(128), 0, st, workspace, nchunks, F, dense ? bias : nullptr, out->vals,
                                                        out->vstride, out->flags, out->fstride);
  EVC_LAUNCH_CHECK("linear_reduce");
  return EVC_OK;
}

int64_t evc_bin_events_workspace(int64_t n, int32_t H, int32_t W, int32_t bins) {
  (void)bins;
  if (n < 1) n = 1;
  const int end_bit = bits_for((uint32_t)(2 * H * W));
  return (int64_t)(4 * align256(n * 4) + align256(cub_temp_bytes(n, end_bit)));
}

int evc_bin_events(const uint64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t lo, int64_t hi,
                   int64_t tau, int64_t delta, int32_t H, int32_t W, int32_t kind, int32_t bins, float* out,
                   void* workspace, int64_t workspace_bytes, void* stream) {
  EVC_CHECK_ARG(out && H > 0 && W > 0 && delta > 0, "bin_events: bad argument");
  EVC_CHECK_ARG(kind >= 0 && kind <= 2, "bin_events: unknown encoder");
  EVC_CHECK_ARG(kind != EVC_ENC_VOXEL || (bins >= 1 && bins <= 32), "bin_events: voxel bins must be in [1, 32]");
  const int C = kind == EVC_ENC_VOXEL ? bins : 2;
  cudaStream_t st = as_stream(stream);
  cudaError_t err = cudaMemsetAsync(out, 0, sizeof(float) * (size_t)C * H * W, st);
  if (err != cudaSuccess) {
    set_error(std::string("evc: bin_events memset: ") + cudaGetErrorString(err));
    return EVC_ECUDA;
  }
  const int64_t n64 = hi - lo;
  if (n64 <= 0) return EVC_OK;
  EVC_CHECK_ARG(n64 < (1LL << 31), "bin_events: window too large");
  EVC_CHECK_ARG(t && x && y && p && workspace, "bin_events: null event column");
  const int n = (int)n64;
  const int end_bit = bits_for((uint32_t)(2 * H * W));
  const size_t need = (size_t)evc_bin_events_workspace(n, H, W, bins);
  if ((size_t)workspace_bytes < need) {
    set_error("evc: bin_events workspace too small");
    return EVC_ENOSPC;
  }
  char* ws = static_cast<char*>(workspace);
  const size_t a = align256((size_t)n * 4);
  uint32_t* k_in = reinterpret_cast<uint32_t*>(ws);
  uint32_t* k_out = reinterpret_cast<uint32_t*>(ws + a);
  int32_t* v_in = reinterpret_cast<int32_t*>(ws + 2 * a);
  int32_t* v_out = reinterpret_cast<int32_t*>(ws + 3 * a);
  void* temp = ws + 4 * a;
  size_t temp_bytes = cub_temp_bytes(n, end_bit);
  launch_pdl(k_event_keys, dim3(cdiv(n, 256)), dim3(256), 0, st, x, y, p, lo, n, H, W, kind, k_in, v_in);
  EVC_LAUNCH_CHECK("event_keys");
  err = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, n, 0, end_bit, st);
  if (err != cudaSuccess) {
    set_error(std::string("evc: bin_events sort: ") + cudaGetErrorString(err));
    return EVC_ECUDA;
  }
  launch_pdl(k_event_runs, dim3(cdiv(n, 256)), dim3(256), 0, st, t, p, k_out, v_out, n, tau - delta, delta, H * W, kind, bins, out);
  EVC_LAUNCH_CHECK("event_runs");
  return EVC_OK;
}

}  // extern "C"

namespace evc {
int init_linear_events() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_linear_partial) != cudaSuccess) return EVC_ECUDA;
  return EVC_OK;
}
}  // namespace evc
