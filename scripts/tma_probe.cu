// Minimal TMA bring-up probe: encodes tensor maps of increasing complexity and
// loads one box each.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe scripts/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int nbytes, int x, int y, int c) {
  __shared__ __align__(1024) float buf[32 * 32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(nbytes) : "memory");
    if (RANK == 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
              "r"(sbuf),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(y), "r"(sbar)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
          "[%6];" ::"r"(sbuf),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(y), "r"(c), "r"(0), "r"(sbar)
          : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(sbar)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiled enc = (EncodeTiled)p;
  printf("encoder %p q=%d\n", p, (int)q);
  float *g, *out;
  cudaMalloc(&g, 8 * 16 * 32 * 4);
  cudaMalloc(&out, 32 * 32 * 4);
  struct Case {
    const char* name;
    int rank;
    CUtensorMapSwizzle sw;
    cuuint32_t box2;
    int x, y, c;
  } cases[] = {{"2d none", 2, CU_TENSOR_MAP_SWIZZLE_NONE, 0, 0, 0, 0},
               {"2d sw128", 2, CU_TENSOR_MAP_SWIZZLE_128B, 0, 0, 0, 0},
               {"2d sw128 x=-1", 2, CU_TENSOR_MAP_SWIZZLE_128B, 0, -1, 0, 0},
               {"2d sw128 y=-1", 2, CU_TENSOR_MAP_SWIZZLE_128B, 0, 0, -1, 0},
               {"4d none box C=8 at 0", 4, CU_TENSOR_MAP_SWIZZLE_NONE, 8, 0, 0, 0},
               {"4d sw128 box C=8 at 0", 4, CU_TENSOR_MAP_SWIZZLE_128B, 8, 0, 0, 0},
               {"4d sw128 box C=8 x=-1", 4, CU_TENSOR_MAP_SWIZZLE_128B, 8, -1, 3, 0},
               {"4d sw128 box C=32>dim", 4, CU_TENSOR_MAP_SWIZZLE_128B, 32, 0, 0, 0},
               {"4d sw128 box C=32 c=16", 4, CU_TENSOR_MAP_SWIZZLE_128B, 32, -1, -1, 0}};
  int ci = -1;
  for (auto& c : cases) {
    ++ci;
    if (only >= 0 && ci != only) continue;
    CUtensorMap m;
    CUresult r;
    int nbytes;
    if (c.rank == 2) {
      cuuint64_t dims[2] = {32, 128}, str[1] = {128};
      cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      nbytes = 32 * 32 * 4;
    } else {
      cuuint64_t dims[4] = {32, 16, 8, 1}, str[3] = {128, 2048, 16384};
      cuuint32_t box[4] = {32, 1, c.box2, 1}, es[4] = {1, 1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      nbytes = 32 * c.box2 * 4;
    }
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", c.name, (int)r);
      continue;
    }
    if (c.rank == 2)
      probe<2><<<1, 128>>>(m, out, nbytes, c.x, c.y, 0);
    else
      probe<4><<<1, 128>>>(m, out, nbytes, c.x, c.y, c.c);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s: %s\n", c.name, cudaGetErrorString(e));
    fflush(stdout);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
