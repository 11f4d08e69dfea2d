// umma_probe.cu -- standalone check of the tcgen05 building blocks used by
// csrc/mma.cu (debug tool, not part of libsable.so).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 8;

__device__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// variant: 0 = tcgen05.st/ld only; 1 = A K-major; 2 = A MN-major
__global__ void probe(const float* A, const float* B, float* D, int variant, int mode) {
  __shared__ __align__(1024) float a[M * K];
  __shared__ __align__(1024) float b[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // fill: A (m, kk), B (n, kk)
  for (int i = tid; i < M * K; i += 128) {
    int m = i / K, kk = i % K;
    int off;
    if (variant == 2) off = ((m >> 2) * 128 + kk * 16 + (m & 3) * 4) >> 2;          // MN-major
    else off = ((m >> 3) * 256 + (m & 7) * 16 + (kk >> 2) * 128 + (kk & 3) * 4) >> 2;  // K-major, LBO 128, SBO 256
    a[off] = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    int n = i / K, kk = i % K;
    b[((n >> 3) * 256 + (n & 7) * 16 + (kk >> 2) * 128 + (kk & 3) * 4) >> 2] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t t = tm;
  if (variant == 0) {
    uint32_t v = __float_as_uint(7.0f + tid);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t + ((warp * 32) << 16)), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  } else if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((variant == 2 ? 1u : 0u) << 15) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint64_t da = variant == 2 ? sdesc(su32(a), mode ? 128 : 4096, mode ? 4096 : 128) : sdesc(su32(a), 128, 256);
    uint64_t db = sdesc(su32(b), 128, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(t), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  if (variant != 0) {
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __syncwarp();
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(t + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < 32; ++n) D[tid * 32 + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  float hA[M * K], hB[N * K], hD[M * 32], R[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (float)(rand() % 5);
  for (int i = 0; i < N * K; ++i) hB[i] = (float)(rand() % 5);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[n * K + k];
      R[m * N + n] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  int cases[][2] = {{0, 0}, {1, 0}, {2, 0}, {2, 1}};
  for (auto& c : cases) {
    cudaMemset(dD, 0, sizeof hD);
    probe<<<1, 128>>>(dA, dB, dD, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0;
    if (c[0] == 0) {
      for (int m = 0; m < M; ++m) err = fmax(err, fabs(hD[m * 32] - (7.0 + m)));
    } else {
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) err = fmax(err, fabs(hD[m * 32 + n] - R[m * N + n]));
    }
    printf("variant %d mode %d: %s max err %g D[0][0..3] %g %g %g %g  R %g %g %g %g  D[5][7] %g R %g\n", c[0], c[1],
           cudaGetErrorString(e), err, hD[0], hD[1], hD[2], hD[3], R[0], R[1], R[2], R[3], hD[5 * 32 + 7], R[5 * N + 7]);
  }
  return 0;
}
