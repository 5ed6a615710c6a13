// Do IMAD, IDP4A / IDP2A, FFMA and DFMA issue to separate pipes? Dependent-free
// streams of each alone and of pairs interleaved, timed with CUDA events;
// reported as thread-ops per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
template <int A, int B>  // 0 none, 1 IMAD, 2 IDP4A, 3 IDP2A, 4 FFMA, 5 DFMA
__global__ void kern(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[ILP], e[ILP], b = seed * 3u + threadIdx.x, c = seed ^ 0x9e37u;
  float fa[ILP], fc = 1.0000001f, fb = 1e-9f;
  double da[ILP], dc = 1.0000000001, db = 1e-12;
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    a[i] = threadIdx.x + i;
    e[i] = threadIdx.x * 7 + i;
    fa[i] = (float)(threadIdx.x + i);
    da[i] = (double)(threadIdx.x + i);
  }
  auto op = [&](int k, int i) {
    if (k == 1) a[i] = a[i] * b + c;
    if (k == 2) e[i] = __dp4a(b, c, e[i]);
    if (k == 3) e[i] = __dp2a_lo(b, c, e[i]);
    if (k == 4) fa[i] = fmaf(fa[i], fc, fb);
    if (k == 5) da[i] = fma(da[i], dc, db);
  };
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        op(A, i);
        op(B, i);
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i] + e[i] + __float_as_uint(fa[i]) + (uint32_t)__double_as_longlong(da[i]);
  if (s == 0x12345678u) out[0] = s;
}

template <int A, int B>
void run(const char* name, const cudaDeviceProp& p, uint32_t* out) {
  const int grid = p.multiProcessorCount * 8, block = 256, iters = (A == 5 || B == 5) ? 512 : 2048;
  kern<A, B><<<grid, block>>>(out, iters, 1);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<A, B><<<grid, block>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * grid * block * (double)iters * 16 * ILP * ((A ? 1 : 0) + (B ? 1 : 0));
  const double clk = p.clockRate * 1e3;
  printf("%-14s %7.1f thread-ops/SM/clk\n", name, ops / (ms * 1e-3) / p.multiProcessorCount / clk);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  uint32_t* out;
  cudaMalloc(&out, 4);
  run<1, 0>("imad", p, out);
  run<2, 0>("idp4a", p, out);
  run<3, 0>("idp2a", p, out);
  run<4, 0>("ffma", p, out);
  run<5, 0>("dfma", p, out);
  run<1, 2>("imad+idp4a", p, out);
  run<1, 3>("imad+idp2a", p, out);
  run<1, 4>("imad+ffma", p, out);
  run<1, 5>("imad+dfma", p, out);
  run<2, 4>("idp4a+ffma", p, out);
  return 0;
}
