// stream_probe.cu -- what the unit executor's access structure can reach
// (not product code).  One-warp CTAs, 32 resident per SM
// at 64 registers, each walking `upc` consecutive "units" of 8 rows x wq
// 16-byte vectors (contiguous), 8 predicated ld.global.cs.v4 per lane per
// unit, all issued before the first add -- the dense part's loads of
// unit_kernel without descriptors, x maps, x, folds or remainder -- then an
// optional dependent FMA chain of `delay` instructions per unit standing in
// for the unit's arithmetic.  Prints GB/s per configuration.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld_cs_if(float4& v, const float4* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];\n}"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
      : "l"(p), "r"((int)pred));
}

__global__ void __launch_bounds__(32, 32)
    stream(const float4* __restrict__ p, long long nunits, int upc, int wq, int delay, float* out) {
  const int lane = threadIdx.x;
  const long long u0 = (long long)blockIdx.x * upc;
  float acc = 0.f;
  for (int i = 0; i < upc; ++i) {
    const long long u = u0 + i;
    if (u >= nunits) break;
    const float4* base = p + u * 8 * wq + lane;
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) ld_cs_if(v[k], base + (long long)k * wq, lane < wq);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    for (int d = 0; d < delay; ++d) acc = fmaf(acc, 1.0000001f, 1e-9f);  // dependent chain
  }
  if (acc == 12345.678f) out[blockIdx.x] = acc;
}

int main() {
  const long long bytes = 343ll << 20;
  float4* p;
  float* out;
  float* scrub;
  const size_t scrub_n = (512ll << 20) / 4;
  cudaMalloc(&p, bytes + (1 << 20));
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&scrub, scrub_n * 4);
  cudaMemset(p, 0, bytes + (1 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int wqs[] = {19, 32};
  const int upcs[] = {1, 3, 4, 16};
  const int delays[] = {0, 64, 128, 256, 512};
  for (int wq : wqs)
    for (int upc : upcs)
      for (int delay : delays) {
        const long long nunits = bytes / (8ll * wq * 16);
        const unsigned grid = (unsigned)((nunits + upc - 1) / upc);
        float best = 1e9f, sum = 0.f;
        const int reps = 12;
        for (int r = 0; r < reps + 2; ++r) {
          cudaMemsetAsync(scrub, r, scrub_n * 4);  // L2 flush (512 MiB write)
          cudaEventRecord(a);
          stream<<<grid, 32>>>(p, nunits, upc, wq, delay, out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r >= 2) {
            sum += ms;
            best = ms < best ? ms : best;
          }
        }
        const double gb = (double)nunits * 8 * wq * 16 / 1e9;
        printf("wq=%d upc=%d delay=%d units=%lld grid=%u mean %.4f ms %.0f GB/s best %.4f ms %.0f GB/s\n",
               wq, upc, delay, nunits, grid, sum / reps, gb / (sum / reps * 1e-3), best,
               gb / (best * 1e-3));
        fflush(stdout);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
