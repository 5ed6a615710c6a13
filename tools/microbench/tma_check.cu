// Standalone check of the TMA staging helpers (csrc/tma.cuh): one CTA loads a
// box of a u16 image at several (possibly out-of-image) origins and compares
// it with the image (zero outside). Exit code 0 = all boxes identical.
// Measured on B200: the box's inner start coordinate must be a multiple of 16
// bytes (x % 8 == 0 for u16); an unaligned x faults with "illegal instruction".
// Callers align the start down and widen the box (refine.cu).
#include <cstdio>
#include <vector>

#include "../../paper_1905_06228_b200/csrc/tma.cuh"

using namespace dicb200;

struct alignas(64) One {
  CUtensorMap m;
};

__global__ void k(const __grid_constant__ One tm, int x, int y, int bw, int bh, uint16_t* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  unsigned char* dst = sm + ((128u - (tma_smem_u32(sm) & 127u)) & 127u);
  if (threadIdx.x == 0) {
    tma_mbar_init(&bar, 1);
    tma_mbar_expect_tx(&bar, (uint32_t)(bw * bh * 2));
    tma_load_2d(dst, &tm.m, x, y, &bar);
  }
  __syncthreads();
  tma_mbar_wait(&bar, 0);
  const uint16_t* s = reinterpret_cast<const uint16_t*>(dst);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = s[i];
}

int main() {
  const int W = 128, H = 96, bw = 88, bh = 53;
  std::vector<uint16_t> img(W * H);
  for (int i = 0; i < W * H; ++i) img[i] = (uint16_t)(i * 7 + 1);
  uint16_t *dimg, *dout;
  cudaMalloc(&dimg, img.size() * 2);
  cudaMalloc(&dout, bw * bh * 2);
  cudaMemcpy(dimg, img.data(), img.size() * 2, cudaMemcpyHostToDevice);
  One tm;
  if (!tma_encode_2d(&tm.m, dimg, 2, W, H, W, bw, bh)) {
    printf("encode failed\n");
    return 2;
  }
  int bad = 0;
  const int org[7][2] = {{0, 7}, {8, 0}, {-8, 0}, {0, -7}, {-8, -7}, {48, 50}, {-16, 60}};
  for (auto& o : org) {
    k<<<1, 128, bw * bh * 2 + 128>>>(tm, o[0], o[1], bw, bh, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("origin (%d,%d): %s\n", o[0], o[1], cudaGetErrorString(e));
      cudaDeviceReset();
      cudaMalloc(&dimg, img.size() * 2);
      cudaMalloc(&dout, bw * bh * 2);
      cudaMemcpy(dimg, img.data(), img.size() * 2, cudaMemcpyHostToDevice);
      tma_encode_2d(&tm.m, dimg, 2, W, H, W, bw, bh);
      ++bad;
      continue;
    }
    std::vector<uint16_t> got(bw * bh);
    cudaMemcpy(got.data(), dout, got.size() * 2, cudaMemcpyDeviceToHost);
    int mism = 0;
    for (int yy = 0; yy < bh; ++yy)
      for (int xx = 0; xx < bw; ++xx) {
        const int gx = o[0] + xx, gy = o[1] + yy;
        const uint16_t exp = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? img[gy * W + gx] : 0;
        mism += got[yy * bw + xx] != exp;
      }
    printf("origin (%d,%d): %d mismatches\n", o[0], o[1], mism);
    bad += mism != 0;
  }
  return bad;
}
