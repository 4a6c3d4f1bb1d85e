// The NS epilogue's store pattern in isolation: 8 warps per CTA, each writes a 32-row x 32-column BF16
// chunk as 8 iterations of (8 lanes x 8 B contiguous per row, 4 rows per instruction) into a row-major
// matrix of pitch `ld` elements; one CTA per SM, each on its own 128 x 128 tile.  Reports ns per chunk.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>   // 0: stores only; 1: each store fed by an LDS.128 of a staged 32 x 32 FP32 chunk (the NS row pass);
                     // 2: as 1 plus an FP32 float4 store per group (update phases)
__global__ void __launch_bounds__(256, 1) k(uint2* __restrict__ out, int ld, int reps, unsigned long long* t,
                                            float* __restrict__ fout) {
  __shared__ float4 Sw[8][32 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rsub = lane >> 3, q4 = lane & 7;
  for (int e = lane; e < 256; e += 32) Sw[warp][e] = make_float4(e, warp, 1.f, 2.f);
  __syncwarp();
  const int row0 = (warp & 3) * 32, col0 = (warp >> 2) * 64;
  uint2* base = out + (size_t)blockIdx.x * 128 * ld / 4;   // this CTA's 128-row band (ld bf16 = ld / 4 uint2)
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int r = 0; r < reps; ++r)
    for (int c = 0; c < 2; ++c) {
#pragma unroll 4
      for (int it = 0; it < 8; ++it) {
        const int i = row0 + 4 * it + rsub, j = col0 + c * 32 + 4 * q4;
        if (MODE == 0) {
          base[((size_t)i * ld + j) / 4] = make_uint2(i * 7 + r, j + c);
        } else {
          const int rr = 4 * it + rsub;
          const float4 a = Sw[warp][rr * 8 + (q4 ^ (rr & 7))];
          const float o0 = -a.x, o1 = -a.y, o2 = -a.z, o3 = -a.w + (float)r;
          __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
          base[((size_t)i * ld + j) / 4] = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          if (MODE == 2)
            reinterpret_cast<float4*>(fout)[((size_t)blockIdx.x * 128 * ld + (size_t)i * ld + j) / 4] = make_float4(o0, o1, o2, o3);
        }
      }
      __syncwarp();
    }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}

int main() {
  const int ld = 512;   // bf16 elements per row (1 KB)
  uint2* out;
  cudaMalloc(&out, (size_t)148 * 128 * ld * 2);
  unsigned long long* t;
  cudaMalloc(&t, 8 * 148);
  float* fout;
  cudaMalloc(&fout, (size_t)148 * 128 * ld * 4);
  auto runk = [&](auto kern, int ctas, const char* name) {
    const int reps = 200;
    kern<<<ctas, 256>>>(out, ld, 10, t, fout);
    kern<<<ctas, 256>>>(out, ld, reps, t, fout);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, t, 8 * ctas, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < ctas; ++i) s += (double)h[i] / ctas;
    printf("%-28s ctas %3d: %.1f ns per 32x32 chunk per warp (%s)\n", name, ctas, s / (reps * 2), cudaGetErrorString(cudaGetLastError()));
  };
  for (int ctas : {1, 148}) {
    runk(k<0>, ctas, "bf16 stores");
    runk(k<1>, ctas, "LDS + bf16 stores");
    runk(k<2>, ctas, "LDS + bf16 + fp32 stores");
  }
}
