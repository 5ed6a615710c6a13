// Feasibility probe for a tensor-core ZNCC search: tcgen05.mma kind::i8
// (u8 x u8 -> s32, exact) with
//   A (M=128 positions = 16 x-offsets x 8 y-offsets, MN-major, no swizzle) read
//     straight out of a "16-px window" image layout T[X][y][16] with
//     SBO = 16 B (next y) and LBO = H*16 B (next X), i.e. overlapping core
//     matrices: A[(mx,my)][k=(j,i)] = img[my + rg*8 + i][mx + cg*4 + j];
//   B (N templates, K-major, no swizzle) in MMA order.
// Checks D[(mx,my)][n] = sum_{r<48,c<44} img[my+r][mx+c] * tmpl[n][r][c] exactly
// and times the MMA stream for several N.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int H = 56;      // rows of T (8 + 48)
constexpr int NX = 44;     // X columns of T (11 groups of 4)
constexpr int RG = 6, CG = 11;
constexpr int T_BYTES = NX * H * 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // base offset 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)            // D = s32
         | (0u << 7)          // A = u8
         | (0u << 10)         // B = u8
         | (1u << 15)         // A MN-major
         | (0u << 16)         // B K-major
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

template <int N>
__host__ __device__ constexpr int nblk() { return (RG * CG * 32 * N + T_BYTES) <= 200 * 1024 ? RG * CG : 16; }

template <int N>
__host__ __device__ constexpr int tcols() { return N * 4 <= 32 ? 32 : N * 4 <= 64 ? 64 : N * 4 <= 128 ? 128 : N * 4 <= 256 ? 256 : 512; }

template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) probe(const uint8_t* __restrict__ img, const uint8_t* __restrict__ bmma,
                                                int32_t* __restrict__ out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* T = sm;
  uint8_t* B = sm + T_BYTES;
  __shared__ uint64_t mbar;
  __shared__ uint64_t mbar2;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // T[X][y][i] = img[y][X + i]   (img is 64 wide)
  for (int e = tid; e < NX * H * 16; e += blockDim.x) {
    const int i = e & 15, y = (e >> 4) % H, X = (e >> 4) / H;
    T[e] = img[y * 64 + X + i];
  }
  for (int e = tid; e < nblk<N>() * 32 * N; e += blockDim.x) B[e] = bmma[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(&tmem_base)), "r"(tcols<N>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(&mbar)), "r"(MODE == 7 ? 2 : 1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&mbar2)));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = idesc_i8(128, N);
  if (tid == 0 || (MODE == 7 && tid == 32)) {
    const int wsel = tid >> 5;
    const uint32_t tb = smem_u32(T), bb = smem_u32(B);
    // descriptors: only the start-address field (bits 0..13, 16-B units) changes per MMA
    uint64_t da0;
    if (MODE <= 1 || MODE >= 5) da0 = sdesc(tb, H * 16, 16);
    else if (MODE == 2) da0 = sdesc(tb, 128, 256);
    else if (MODE == 3) da0 = sdesc(tb, 16, 1024) | (2ull << 61);
    else da0 = sdesc(tb, 4096, 1024) | (2ull << 61);
    const uint64_t db0 = sdesc(bb, 128, 256);
    const uint32_t id = (MODE == 2 || MODE == 3) ? (idesc & ~(1u << 15)) : idesc;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int rg = 0; rg < RG; ++rg)
#pragma unroll
        for (int cg = 0; cg < CG; ++cg) {
          uint32_t aoff, boff;
          if (MODE == 0 || MODE >= 5) aoff = (uint32_t)((cg * 4 * H + rg * 8) * 16);
          else if (MODE == 1) aoff = 0;
          else if (MODE == 2) aoff = (uint32_t)(((rg * CG + cg) % 8) * 4096);
          else if (MODE == 3) aoff = (uint32_t)(((rg * CG + cg) % 2) * 16384 + (cg % 4) * 32);
          else aoff = (uint32_t)(((rg * CG + cg) % 8) * 4096);
          boff = MODE == 1 ? 0u : (uint32_t)(((rg * CG + cg) % nblk<N>()) * 32 * N);
          if (MODE == 12) {  // exact bfs_tc stage layout: 4 stages x (T 2 planes 16 rows | B at +24704), 22 MMAs per stage
            const int stage = (rep * RG + rg) & 3;
            const uint32_t sb = tb + (uint32_t)(stage * 41984);
            if (sb + 41984 <= tb + 200 * 1024) {
              const uint64_t dA = sdesc(sb, 256, 16) + (uint64_t)(cg * 64);
              const uint64_t dB = sdesc(sb + 24704, 128, 256) + (uint64_t)(cg * N * 2);
              mma_i8(tmem, dA, dB, id, (rg | cg) != 0);
              mma_i8(tmem + (uint32_t)N, dA + (uint64_t)(11264 >> 4), dB, id, (rg | cg) != 0);
            }
          } else if (MODE == 11) {  // tile structure: D alternates between two buffers per rep, cleared at tile start
            mma_i8(tmem + (uint32_t)((rep & 1) * N), da0 + (aoff >> 4), db0 + (boff >> 4), id, (rg | cg) != 0);
          } else if (MODE == 10) {
            const uint64_t dA = sdesc(tb, 16 * 16, 16) + (uint64_t)(cg * 4 * 16);
            mma_i8(tmem, dA, db0 + (boff >> 4), id, (rep | rg | cg) != 0);
          } else if (MODE == 8 || MODE == 9) {
            mma_i8(tmem, da0 + (aoff >> 4), db0 + (boff >> 4), id, (rep | rg | cg) != 0);
            if (cg == CG - 1) {
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                           :: "r"(smem_u32(&mbar2)) : "memory");
              if (MODE == 9) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            }
          } else if (MODE == 7) {
            if ((rg & 1) == wsel)
              mma_i8(tmem + (uint32_t)(wsel * N), da0 + (aoff >> 4), db0 + (boff >> 4), id, (rep | (rg >> 1) | cg) != 0);
          } else if (MODE >= 5) {
            constexpr int NACC = MODE == 5 ? 2 : 4;
            const int q = (rg * CG + cg) % NACC;
            mma_i8(tmem + (uint32_t)(q * N), da0 + (aoff >> 4), db0 + (boff >> 4), id, (rep | (rg * CG + cg) / NACC) != 0);
          } else
          mma_i8(tmem, da0 + (aoff >> 4), db0 + (boff >> 4), id, (rep | rg | cg) != 0);
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 :: "r"(smem_u32(&mbar)) : "memory");
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\t"
                   "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // D row m = lane m: warp w reads lanes 32w..32w+31
  if (blockIdx.x == 0) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) out[tid * N + c0 + j] = (int32_t)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem), "r"(tcols<N>()));
}

template <int N>
void run(const std::vector<uint8_t>& img, const std::vector<uint8_t>& tmpl) {
  // B in MMA order: block (rg,cg) = N x 32 bytes K-major, core matrices 8 n x 16 k,
  // LBO = 128 B (k half), SBO = 256 B (next 8 n). k = j*8 + i  <->  c = cg*4 + j, r = rg*8 + i
  std::vector<uint8_t> bm((size_t)RG * CG * 32 * N, 0);
  for (int rg = 0; rg < RG; ++rg)
    for (int cg = 0; cg < CG; ++cg)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < 32; ++k) {
          const int j = k / 8, i = k % 8, r = rg * 8 + i, c = cg * 4 + j;
          const size_t off = (size_t)(rg * CG + cg) * 32 * N + (n % 8) * 16 + (n / 8) * 256 + (k / 16) * 128 + (k % 16);
          bm[off] = tmpl[((size_t)n * 48 + r) * 44 + c];
        }
  uint8_t *dimg, *db;
  int32_t* dout;
  CK(cudaMalloc(&dimg, img.size()));
  CK(cudaMalloc(&db, bm.size()));
  CK(cudaMalloc(&dout, 128 * N * 4));
  CK(cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bm.data(), bm.size(), cudaMemcpyHostToDevice));
  const int smem = T_BYTES + nblk<N>() * 32 * N;
  CK(cudaFuncSetAttribute(probe<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 11>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<N, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  probe<N, 0><<<1, 128, smem>>>(dimg, db, dout, 1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> got(128 * N);
  CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  if (nblk<N>() == RG * CG)
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      const int mx = m % 16, my = m / 16;
      int64_t s = 0;
      for (int r = 0; r < 48; ++r)
        for (int c = 0; c < 44; ++c) s += (int64_t)img[(my + r) * 64 + mx + c] * tmpl[((size_t)n * 48 + r) * 44 + c];
      if (s != got[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d got %d want %lld\n", m, n, got[m * N + n], (long long)s);
        ++bad;
      }
    }
  // throughput: 148 x k CTAs, many reps
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 200, grid = 148;
  printf("smem %d\n", smem);
  for (int mode = 0; mode < 13; ++mode) {
  if (mode >= 1 && mode <= 11) continue;
  const int smem_used = mode == 12 ? 200 * 1024 : smem;
  auto k = mode == 0 ? probe<N, 0> : mode == 1 ? probe<N, 1> : mode == 2 ? probe<N, 2> : mode == 3 ? probe<N, 3> : mode == 4 ? probe<N, 4> : mode == 5 ? probe<N, 5> : mode == 6 ? probe<N, 6> : mode == 7 ? probe<N, 7> : mode == 8 ? probe<N, 8> : mode == 9 ? probe<N, 9> : mode == 10 ? probe<N, 10> : mode == 11 ? probe<N, 11> : probe<N, 12>;
  k<<<grid, 128, smem_used>>>(dimg, db, dout, 4);
  cudaEventRecord(a);
  k<<<grid, 128, smem_used>>>(dimg, db, dout, reps);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("mode %d: ", mode);
  const double mmas = (double)grid * reps * RG * CG * (mode == 12 ? 2 : 1);
  const double macs = mmas * 128.0 * N * 32;
  printf("N=%3d exact=%s (bad %ld)  %.3f ms  %.1f clk/MMA/SM  %.1f TMAC/s (i8)\n", N, bad ? "NO" : "yes", bad, ms,
         ms * 1e-3 * 1.965e9 / (mmas / grid), macs / (ms * 1e-3) / 1e12);
  }
  cudaFree(dimg);
  cudaFree(db);
  cudaFree(dout);
}

int main() {
  std::vector<uint8_t> img(64 * 64);
  srand(1);
  for (auto& v : img) v = (uint8_t)(rand() & 255);
  std::vector<uint8_t> tmpl(256 * 48 * 44, 0);
  for (int n = 0; n < 256; ++n)
    for (int r = 0; r < 41; ++r)
      for (int c = 0; c < 41; ++c) tmpl[((size_t)n * 48 + r) * 44 + c] = (uint8_t)(rand() & 255);
  run<16>(img, tmpl);
  run<32>(img, tmpl);
  run<48>(img, tmpl);
  run<64>(img, tmpl);

  return 0;
}
