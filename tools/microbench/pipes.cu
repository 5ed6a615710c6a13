// Pipe-rate microbenchmark for the roofline denominators of the search kernels:
// dependent-free IMAD, IDP4A, FFMA, DFMA, IADD3 streams, timed with CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
template <int OP>
__global__ void kern(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[ILP], b = seed * 3u + threadIdx.x, c = seed ^ 0x9e37u;
  float fa[ILP], fb = (float)b * 1e-9f, fc = 1.0000001f;
  double da[ILP], db = (double)b * 1e-12, dc = 1.0000000001;
  #pragma unroll
  for (int i = 0; i < ILP; ++i) { a[i] = threadIdx.x + i; fa[i] = (float)(threadIdx.x + i); da[i] = (double)(threadIdx.x + i); }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int u = 0; u < 16; ++u) {
      #pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (OP == 0) a[i] = a[i] * b + c;                         // IMAD
        if (OP == 1) a[i] = __dp4a(b, c, a[i]);                   // IDP4A (u8x4 as signed here)
        if (OP == 2) fa[i] = fmaf(fa[i], fc, fb);                 // FFMA
        if (OP == 3) da[i] = fma(da[i], dc, db);                  // DFMA
        if (OP == 4) a[i] = __byte_perm(a[i], b, 0x5432) ^ c;      // PRMT+LOP
        if (OP == 5) { uint32_t r; asm volatile("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(c), "r"(a[i])); a[i] = r; }
      }
    }
  }
  uint32_t s = 0;
  #pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i] + __float_as_uint(fa[i]) + (uint32_t)__double_as_longlong(da[i]);
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, p.multiProcessorCount, p.clockRate);
  uint32_t* out; cudaMalloc(&out, 4);
  const char* names[] = {"imad", "idp4a_s8", "ffma", "dfma", "prmt_lop", "idp4a_u8"};
  const int iters = 4096;
  for (int op = 0; op < 6; ++op) {
    for (int blocks_per_sm : {8}) {
      int grid = p.multiProcessorCount * blocks_per_sm, block = 256;
      auto launch = [&]() {
        switch (op) {
          case 0: kern<0><<<grid, block>>>(out, iters, 1); break;
          case 1: kern<1><<<grid, block>>>(out, iters, 1); break;
          case 2: kern<2><<<grid, block>>>(out, iters, 1); break;
          case 3: kern<3><<<grid, block>>>(out, iters / 8, 1); break;
          case 4: kern<4><<<grid, block>>>(out, iters, 1); break;
          case 5: kern<5><<<grid, block>>>(out, iters, 1); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = 5.0 * grid * block * (double)(op == 3 ? iters / 8 : iters) * 16 * ILP;
      printf(", \"%s_Ginstr_per_s\": %.1f", names[op], ops / (ms * 1e-3) / 1e9);
    }
  }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
