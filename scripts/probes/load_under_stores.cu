// Standalone probe (not part of the library): latency of a dependent L2-hit
// load while the SMs stream 128-bit stores to HBM (K3's situation at cfg3:
// a tile's bin -> supports -> table rows chain runs beside the stores of the
// other resident CTAs).
// Each CTA: lane 0 of warp 0 chases pointers through a 1 MiB (L2-resident)
// ring of uint4 {next, ...}; the other warps store 2 x float4 per thread per
// iteration until the chaser is done. Reported: mean cycles per chase step,
// split by whether the CTA's SM stores, and the store bandwidth reached.
//   load path  0 ld.global.cg   1 ld.global.nc   2 cp.async (LDGSTS) + wait
//              3 cp.async.bulk + mbarrier (TMA unit)   4 tex1Dfetch
//   storers    0 none   1 every SM   2 even SMs only (odd SMs only chase)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o load_under_stores load_under_stores.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kRing = 65536;   // uint4 entries (1 MiB)
constexpr int kSteps = 96;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

template <int PATH>
__device__ __forceinline__ unsigned chase_step(const uint4* ring, cudaTextureObject_t tex, unsigned idx,
                                               uint4* sbuf, unsigned bar, unsigned& phase) {
  if (PATH == 0) {
    unsigned v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(ring + idx) : "memory");
    return v;
  } else if (PATH == 1) {
    unsigned v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(ring + idx) : "memory");
    return v;
  } else if (PATH == 2) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sbuf)), "l"(ring + idx) : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    return *reinterpret_cast<volatile unsigned*>(sbuf);
  } else if (PATH == 3) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(bar) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
            smem_u32(sbuf)),
        "l"(ring + idx), "r"(bar)
        : "memory");
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar), "r"(phase)
          : "memory");
    }
    phase ^= 1u;
    return *reinterpret_cast<volatile unsigned*>(sbuf);
  } else {
    return tex1Dfetch<uint4>(tex, (int)idx).x;
  }
}

template <int PATH>
__global__ void __launch_bounds__(256, 4)
probe(const uint4* ring, cudaTextureObject_t tex, float4* out, long cta_f4, int storers, long long* res,
      int max_iters) {
  __shared__ volatile int done;
  __shared__ alignas(16) uint4 sbuf;
  __shared__ alignas(8) unsigned long long mbar;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const bool stores = storers == 1 || (storers == 2 && (smid & 1u) == 0u);
  if (threadIdx.x == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      unsigned idx = (blockIdx.x * 7919u) % kRing, phase = 0;
      // a few untimed steps so the store warps are running
      for (int s = 0; s < 8; ++s) idx = chase_step<PATH>(ring, tex, idx, &sbuf, smem_u32(&mbar), phase);
      const long long t0 = clock64();
      for (int s = 0; s < kSteps; ++s) idx = chase_step<PATH>(ring, tex, idx, &sbuf, smem_u32(&mbar), phase);
      const long long t1 = clock64();
      res[blockIdx.x * 4 + 0] = t1 - t0;
      res[blockIdx.x * 4 + 1] = smid;
      res[blockIdx.x * 4 + 3] = idx;
      done = 1;
    }
    return;
  }
  long long iters = 0;
  if (stores) {
    float4* base = out + (long)blockIdx.x * cta_f4;
    const float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int t = threadIdx.x - 32;   // 0..223
    // per iteration the 7 warps store 2 x 3584 B, contiguous per warp store
    for (int it = 0; it < max_iters && !done; ++it) {
      float4* p = base + (long)it * 448 + t;
      __stcs(p, v);
      __stcs(p + 224, v);
      ++iters;
    }
  }
  if (threadIdx.x == 32) res[blockIdx.x * 4 + 2] = iters;
}

template <int PATH>
void run(const char* name, const uint4* ring, cudaTextureObject_t tex, float4* out, long cta_f4, int ctas,
         long long* res_d, int max_iters) {
  std::vector<long long> res(ctas * 4);
  for (int storers = 0; storers < 3; ++storers) {
    cudaMemset(res_d, 0, sizeof(long long) * ctas * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<PATH><<<ctas, 256>>>(ring, tex, out, cta_f4, storers, res_d, max_iters);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(res.data(), res_d, sizeof(long long) * ctas * 4, cudaMemcpyDeviceToHost);
    double cyc_st = 0, cyc_q = 0, bytes = 0;
    int n_st = 0, n_q = 0;
    for (int i = 0; i < ctas; ++i) {
      const bool st = storers == 1 || (storers == 2 && (res[i * 4 + 1] & 1) == 0);
      (st ? cyc_st : cyc_q) += (double)res[i * 4] / kSteps;
      (st ? n_st : n_q) += 1;
      bytes += (double)res[i * 4 + 2] * 7168.0;
    }
    printf("%-22s storers=%d  kernel %.1f us  stores %.0f GB/s  cycles/step: storing SMs %.0f (n=%d)  quiet SMs %.0f (n=%d)\n",
           name, storers, ms * 1e3, bytes / (ms * 1e-3) / 1e9, n_st ? cyc_st / n_st : 0.0, n_st,
           n_q ? cyc_q / n_q : 0.0, n_q);
  }
}

int main() {
  const int ctas = 148 * 4;
  const int max_iters = 512;                 // 3.67 MB per CTA at most
  const long cta_f4 = (long)max_iters * 448;
  float4* out;
  cudaMalloc(&out, sizeof(float4) * cta_f4 * ctas);
  std::vector<uint4> ring(kRing);
  std::vector<unsigned> perm(kRing);
  for (int i = 0; i < kRing; ++i) perm[i] = i;
  srand(1);
  for (int i = kRing - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
  for (int i = 0; i < kRing; ++i) ring[perm[i]] = make_uint4(perm[(i + 1) % kRing], 0, 0, 0);
  uint4* ring_d;
  cudaMalloc(&ring_d, sizeof(uint4) * kRing);
  cudaMemcpy(ring_d, ring.data(), sizeof(uint4) * kRing, cudaMemcpyHostToDevice);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = ring_d;
  rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
  rd.res.linear.sizeInBytes = sizeof(uint4) * kRing;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  long long* res_d;
  cudaMalloc(&res_d, sizeof(long long) * ctas * 4);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>("ld.global.cg", ring_d, tex, out, cta_f4, ctas, res_d, max_iters);
    run<1>("ld.global.nc", ring_d, tex, out, cta_f4, ctas, res_d, max_iters);
    run<2>("cp.async 16B + wait", ring_d, tex, out, cta_f4, ctas, res_d, max_iters);
    run<3>("cp.async.bulk + mbar", ring_d, tex, out, cta_f4, ctas, res_d, max_iters);
    run<4>("tex1Dfetch", ring_d, tex, out, cta_f4, ctas, res_d, max_iters);
  }
  return 0;
}
