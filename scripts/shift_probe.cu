// Probe: can a tcgen05 SW128 K-major smem descriptor start at a row offset that is not a
// multiple of 8 (1024 B)?  D[128x16] = A[shift .. shift+127, 0:32] . B[16, 0:32]^T, A stored once
// in the canonical 128B-swizzled layout (row r, 16B chunk k at chunk k ^ (r & 7)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/shift_probe.bin scripts/shift_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t base_off) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)(base_off & 7) << 49) | ((uint64_t)2 << 61);
}

__global__ void probe(const float* A, const float* B, float* D, int shift, int use_bo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~(uintptr_t)1023);
  float* As = reinterpret_cast<float*>(base);            // 144 rows x 32
  float* Bs = reinterpret_cast<float*>(base + 144 * 128);  // 16 rows x 32
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 144 * 32; i += blockDim.x) {
    const int r = i / 32, e = i % 32, k = e / 4, sub = e % 4;
    As[r * 32 + ((k ^ (r & 7)) * 4) + sub] = A[i];
  }
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
    const int r = i / 32, e = i % 32, k = e / 4, sub = e % 4;
    Bs[r * 32 + ((k ^ (r & 7)) * 4) + sub] = B[i];
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t a0 = su32(As) + shift * 128, b0 = su32(Bs);
    const uint32_t bo = use_bo ? ((a0 >> 7) & 7) : 0;
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t da = desc(a0 + kk * 32, bo), db = desc(b0 + kk * 32, 0);
      const uint32_t acc = kk ? 1u : 0u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(IDESC), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n\t}" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  const uint32_t taddr = tmem + ((uint32_t)(32 * (threadIdx.x / 32)) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) D[threadIdx.x * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(32));
  }
}

int main() {
  float hA[144 * 32], hB[16 * 32], hD[128 * 16];
  for (int i = 0; i < 144 * 32; ++i) hA[i] = (float)((i * 7 + 3) % 11 - 5);
  for (int i = 0; i < 16 * 32; ++i) hB[i] = (float)((i * 5 + 1) % 7 - 3);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int use_bo = 0; use_bo < 2; ++use_bo)
    for (int shift = 0; shift < 9; ++shift) {
      probe<<<1, 128, 64 * 1024>>>(A, B, D, shift, use_bo);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
          double ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)hA[(m + shift) * 32 + k] * hB[n * 32 + k];
          if (hD[m * 16 + n] != (float)ref) ++bad;
        }
      printf("use_base_offset=%d shift=%d: %s, mismatches %d / 2048\n", use_bo, shift, cudaGetErrorString(e), bad);
    }
  return 0;
}
