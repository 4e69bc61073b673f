// Standalone probe (not part of the library): HBM write ceilings on B200 for
// store patterns K3 could use. nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill_stride(float4* out, long n4, int cs) {
  const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    if (cs) __stcs(out + i, v); else out[i] = v;
}

// each CTA writes whole 16 KB tiles (1024 float4), tile = blockIdx + k*gridDim
__global__ void fill_tiles(float4* out, long ntiles, int cs) {
  const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    float4* p = out + t * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
      if (cs) __stcs(p + i, v); else p[i] = v;
  }
}

// TMA bulk store of a zeroed 16 KB shared buffer per tile
__global__ void fill_tma(float4* out, long ntiles) {
  __shared__ alignas(128) float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(buf);
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;"
                   :: "l"(out + t * 1024), "r"(s) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const long bytes = 5368709120L;   // cfg1 output
  float4* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  const long n4 = bytes / 16, ntiles = bytes / 16384;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %8.1f GB/s  (%s)\n", name, bytes * 10 / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int cs = 0; cs < 2; ++cs) {
    char nm[64];
    snprintf(nm, 64, "stride grid=148*16 cs=%d", cs);
    timeit(nm, [&] { fill_stride<<<148 * 16, 256>>>(out, n4, cs); });
    snprintf(nm, 64, "stride grid=148*64 cs=%d", cs);
    timeit(nm, [&] { fill_stride<<<148 * 64, 256>>>(out, n4, cs); });
    snprintf(nm, 64, "tiles16K grid=148*8 cs=%d", cs);
    timeit(nm, [&] { fill_tiles<<<148 * 8, 256>>>(out, ntiles, cs); });
    snprintf(nm, 64, "tiles16K grid=148*32 cs=%d", cs);
    timeit(nm, [&] { fill_tiles<<<148 * 32, 256>>>(out, ntiles, cs); });
  }
  timeit("tma16K grid=148*4", [&] { fill_tma<<<148 * 4, 128>>>(out, ntiles); });
  timeit("tma16K grid=148*8", [&] { fill_tma<<<148 * 8, 128>>>(out, ntiles); });
  return 0;
}
