// bw_probe.cu — HBM read-bandwidth probe for the decode kernel's memory pipeline design.
// (a) plain vectorized LDG streaming; (b) 1-D bulk-async-copy rings (one producer lane per
// page, NCONS consumer warps that only wait + release) for several ring depths / chunk sizes /
// CTAs per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra.uni W_%=;\n}" ::"r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(n), "r"(bar), "l"(pol) : "memory");
}

__global__ void ldg_stream(const int4* __restrict__ a, size_t n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    int4 v0 = __ldcs(a + i), v1 = __ldcs(a + i + st), v2 = __ldcs(a + i + 2 * st), v3 = __ldcs(a + i + 3 * st);
    acc.x ^= v0.x ^ v1.x ^ v2.x ^ v3.x; acc.y ^= v0.y ^ v1.y ^ v2.y ^ v3.y;
  }
  for (; i < n; i += st) { int4 v = __ldcs(a + i); acc.x ^= v.x; }
  if (acc.x == 0x12345678 && acc.y == 7) sink[0] = 1;
}

// ring: S stages of CH bytes; chunk c of this CTA goes to consumer warp c % NCONS
// chunk order of CTA b: mode 0 contiguous range; mode 1 tiles of TP chunks round-robin
// (tile b, b+grid, ...: the decode kernel's static schedule); mode 2 contiguous tile range
__device__ __forceinline__ size_t chunk_of(int mode, size_t j, size_t c0, int TP) {
  if (mode == 1) {
    const size_t t = blockIdx.x + (j / TP) * gridDim.x;
    return t * TP + j % TP;
  }
  return c0 + j;
}
template <int NCONS>
__global__ void ring_stream(const uint8_t* a, size_t nchunks, int CH, int S, int mode, int TP) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = smem_u32(sm);
  const uint32_t bars = base + S * CH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(bars + 8 * s, 1); mbar_init(bars + 8 * (S + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // contiguous range of chunks per CTA
  const size_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const size_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
  const size_t n = c1 > c0 ? c1 - c0 : 0;
  if (warp == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int B = S < 32 ? S : 32;
    for (size_t i0 = 0; i0 < n; i0 += B) {
      const int nb = (int)min((size_t)B, n - i0);
      if (lane < nb) {
        const size_t j = i0 + lane;
        const int s = (int)(j % S);
        mbar_wait(bars + 8 * (S + s), ((j / S) & 1) ^ 1);
        mbar_expect(bars + 8 * s, CH);
        bulk(base + s * CH, a + chunk_of(mode, j, c0, TP) * CH, CH, bars + 8 * s, pol);
      }
      __syncwarp();
    }
  } else {
    const int w = warp - 1;
    for (size_t j = w; j < n; j += NCONS) {
      const int s = (int)(j % S);
      mbar_wait(bars + 8 * s, (j / S) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + 8 * (S + s));
    }
  }
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* a;
  int* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& f) {
    f();
    cudaEventRecord(e0);
    const int R = 5;
    for (int r = 0; r < R; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes / (ms / R * 1e-3) / 1e9;
  };
  for (int bpsm : {4, 8, 16}) {
    double gbs = timeit([&] { ldg_stream<<<sms * bpsm, 256>>>((const int4*)a, bytes / 16, sink); });
    printf("ldg_stream blocks/SM=%d: %.0f GB/s\n", bpsm, gbs);
  }
  for (int mode : {0, 1, 2}) {
    for (int TP : {32, 31, 64}) {
      const int ch = 8192, S = 16;
      const int smem = S * ch + 2 * S * 8 + 64;
      auto k = ring_stream<8>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const size_t nch = (bytes / ch) / (TP * sms) * (TP * sms);
      double gbs = timeit([&] { k<<<sms, 9 * 32, smem>>>(a, nch, ch, S, mode, TP); });
      gbs *= (double)(nch * ch) / bytes;
      printf("ring 8K S=16 mode=%d tile=%d chunks: %.0f GB/s %s\n", mode, TP, gbs,
             cudaGetErrorString(cudaGetLastError()));
      if (mode != 1) break;
    }
  }
  // ring depth sweep (mode 0): bytes in flight per SM vs achieved bandwidth
  for (int S : {8, 16, 24}) {  // multiples of the 8 consumers (a stage is always one warp's)
    const int ch = 8192;
    const int smem = S * ch + 2 * S * 8 + 64;
    auto k = ring_stream<8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const size_t nch = (bytes / ch) / (32 * sms) * (32 * sms);
    double gbs = timeit([&] { k<<<sms, 9 * 32, smem>>>(a, nch, ch, S, 0, 32); });
    gbs *= (double)(nch * ch) / bytes;
    printf("ring 8K S=%d (%d KB in flight/SM): %.0f GB/s %s\n", S, S * 8, gbs, cudaGetErrorString(cudaGetLastError()));
  }
  // per-SM ceiling: fewer CTAs than SMs (config 4 at G = 128 streams on 128 SMs)
  for (int G : {64, 96, 128, 136, 148}) {
    for (int S : {16, 24}) {
      const int ch = 8192;
      const int smem = S * ch + 2 * S * 8 + 64;
      auto k = ring_stream<8>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const size_t nch = (bytes / ch) / (32 * G) * (32 * G);
      double gbs = timeit([&] { k<<<G, 9 * 32, smem>>>(a, nch, ch, S, 0, 32); });
      gbs *= (double)(nch * ch) / bytes;
      printf("ring 8K S=%d grid=%d: %.0f GB/s = %.1f GB/s per CTA\n", S, G, gbs, gbs / G);
    }
  }
  // launch-granular, config 4 size: 268 MB per launch (128 units x 2 MiB)
  for (int G : {128, 148}) {
    const size_t slice = 256ull << 20, nsl = bytes / slice;
    const int ch = 8192, S = 16;
    const int smem = S * ch + 2 * S * 8 + 64;
    auto k = ring_stream<8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEventRecord(e0);
    const int N = 100;
    for (int i = 0; i < N; ++i) k<<<G, 9 * 32, smem>>>(a + (i % nsl) * slice, slice / ch, ch, S, 0, 32);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ring 8K S=16 grid=%d, 268 MB per launch, back-to-back: %.1f us/launch, %.0f GB/s\n", G,
           ms / N * 1e3, slice / (ms / N * 1e-3) / 1e9);
  }
  // launch-granular streaming: back-to-back launches over distinct 537 MB slices (the size of
  // one config-3 layer-step), the ceiling for a kernel that must stream that much per launch
  {
    const size_t slice = 537ull << 20, nsl = bytes / slice;
    const int ch = 8192, S = 16;
    const int smem = S * ch + 2 * S * 8 + 64;
    auto k = ring_stream<8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      const int N = 60;
      for (int i = 0; i < N; ++i)
        k<<<sms, 9 * 32, smem>>>(a + (i % nsl) * slice, slice / ch, ch, S, 0, 32);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("ring 8K S=16, 537 MB per launch, back-to-back: %.1f us/launch, %.0f GB/s\n",
             ms / N * 1e3, slice / (ms / N * 1e-3) / 1e9);
    }
  }
  return 0;
}
