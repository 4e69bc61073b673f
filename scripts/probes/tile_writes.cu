// Standalone probe (not part of the library): HBM write rate of K3's tile
// store pattern on the cfg3 grid [32, 8, 128, 128, 128] fp32 (2.15 GB).
//   tiles32   one CTA per (molecule, channel, 16-slab chunk, 64-row block,
//             32-float z window), K3's CTA order (molecule fastest, then
//             channel, then z window, row block, chunk); per slab each thread
//             stores two float4 half a window apart (K3's 8-voxel slot)
//   tiles128z one CTA per (molecule, channel, chunk, row block) looping over
//             the four z windows (z window outer, slab inner)
//   tiles128s same, slab outer, z window inner (whole 512 B rows per slab)
//   stride    plain grid-stride 128-bit fill (ceiling)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tile_writes tile_writes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int B = 32, C = 8, N = 128;           // molecules, channels, voxels per axis
constexpr long SLAB = (long)N * N;              // floats per y-slab
constexpr long GRID = (long)N * SLAB;           // floats per channel grid

__device__ __forceinline__ void st8(float* p, float4 v) {   // slot: quads kk and kk + 4
  __stcs(reinterpret_cast<float4*>(p), v);
  __stcs(reinterpret_cast<float4*>(p + 16), v);
}

// thread t: row r0 = t / 4 (0..63), slot kk = t % 4 (z floats 4kk.., 16+4kk..)
__global__ void tiles32(float* out) {
  unsigned lin = blockIdx.x;
  const int b = lin % B; lin /= B;
  const int c = lin % C; lin /= C;
  const int zb = lin % 4; lin /= 4;
  const int rb = lin % 2; lin /= 2;
  const int chunk = lin;
  const int r = rb * 64 + threadIdx.x / 4, kk = threadIdx.x % 4;
  float* base = out + ((long)b * C + c) * GRID + (long)chunk * 16 * SLAB + (long)r * N + zb * 32 + 4 * kk;
  const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < 16; ++j) st8(base + j * SLAB, v);
}

template <bool SLAB_OUTER>
__global__ void tiles128(float* out) {
  unsigned lin = blockIdx.x;
  const int b = lin % B; lin /= B;
  const int c = lin % C; lin /= C;
  const int rb = lin % 2; lin /= 2;
  const int chunk = lin;
  const int r = rb * 64 + threadIdx.x / 4, kk = threadIdx.x % 4;
  float* base = out + ((long)b * C + c) * GRID + (long)chunk * 16 * SLAB + (long)r * N + 4 * kk;
  const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (SLAB_OUTER) {
    for (int j = 0; j < 16; ++j)
      for (int zb = 0; zb < 4; ++zb) st8(base + j * SLAB + zb * 32, v);
  } else {
    for (int zb = 0; zb < 4; ++zb)
      for (int j = 0; j < 16; ++j) st8(base + j * SLAB + zb * 32, v);
  }
}

__global__ void stride(float4* out, long n4) {
  const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    __stcs(out + i, v);
}

int main() {
  const long floats = (long)B * C * GRID, bytes = floats * 4;
  float* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, a, e);
    printf("%-12s %8.1f GB/s  %.4f ms  (%s)\n", name, bytes * 20 / (ms / 1e3) / 1e9, ms / 20,
           cudaGetErrorString(cudaGetLastError()));
  };
  const int ctas32 = B * C * 4 * 2 * 8, ctas128 = B * C * 2 * 8;
  timeit("tiles32", [&] { tiles32<<<ctas32, 256>>>(out); });
  timeit("tiles128z", [&] { tiles128<false><<<ctas128, 256>>>(out); });
  timeit("tiles128s", [&] { tiles128<true><<<ctas128, 256>>>(out); });
  timeit("stride", [&] { stride<<<148 * 64, 256>>>(reinterpret_cast<float4*>(out), floats / 4); });
  return 0;
}
