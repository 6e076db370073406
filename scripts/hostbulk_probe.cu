// Probe: does cp.async.bulk (global -> shared) accept a pinned, mapped host address (UVA)?
// And how fast is a coalesced zero-copy read / write of host memory from the SMs?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_bulk(const void* src, float* out, int bytes) {
  __shared__ alignas(128) uint8_t buf[4096];
  __shared__ alignas(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b) : "memory");
  float s = 0.f;
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) s += reinterpret_cast<float*>(buf)[i];
  atomicAdd(out, s);
}
__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  float* h; cudaHostAlloc(&h, 1 << 20, cudaHostAllocDefault);
  for (int i = 0; i < 1024; ++i) h[i] = 1.0f;
  float* o; cudaMalloc(&o, 4); cudaMemset(o, 0, 4);
  k_bulk<<<1, 128>>>(h, o, 4096);
  cudaError_t e = cudaDeviceSynchronize();
  float r = 0; cudaMemcpy(&r, o, 4, cudaMemcpyDeviceToHost);
  printf("bulk from pinned host: %s, sum = %.0f (expect 1024)\n", cudaGetErrorString(e), r);
  // zero-copy bandwidth: 768 KiB host -> device and 512 KiB device -> host, like one layer-step
  uint8_t *hs, *hd, *ds, *dd;
  cudaHostAlloc(&hs, 1 << 22, 0); cudaHostAlloc(&hd, 1 << 22, 0); cudaMalloc(&ds, 1 << 22); cudaMalloc(&dd, 1 << 22);
  cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
  for (int kb : {512, 768, 4096}) {
    size_t n = (size_t)kb * 1024 / 16;
    for (int grid : {16, 148}) {
      for (int w = 0; w < 3; ++w) k_copy<<<grid, 256>>>((uint4*)hs, (uint4*)dd, n);
      cudaEventRecord(a);
      for (int w = 0; w < 20; ++w) k_copy<<<grid, 256>>>((uint4*)hs, (uint4*)dd, n);
      cudaEventRecord(c); cudaEventSynchronize(c);
      float ms; cudaEventElapsedTime(&ms, a, c);
      printf("zero-copy read  %5d KiB grid %3d: %.1f us  %.1f GB/s\n", kb, grid, ms * 1e3 / 20, kb * 1024.0 / (ms / 20 * 1e-3) / 1e9);
      cudaEventRecord(a);
      for (int w = 0; w < 20; ++w) k_copy<<<grid, 256>>>((uint4*)ds, (uint4*)hd, n);
      cudaEventRecord(c); cudaEventSynchronize(c);
      cudaEventElapsedTime(&ms, a, c);
      printf("zero-copy write %5d KiB grid %3d: %.1f us  %.1f GB/s\n", kb, grid, ms * 1e3 / 20, kb * 1024.0 / (ms / 20 * 1e-3) / 1e9);
    }
    cudaEventRecord(a);
    for (int w = 0; w < 20; ++w) cudaMemcpyAsync(dd, hs, (size_t)kb * 1024, cudaMemcpyHostToDevice);
    cudaEventRecord(c); cudaEventSynchronize(c);
    float ms; cudaEventElapsedTime(&ms, a, c);
    printf("memcpy H2D      %5d KiB: %.1f us\n", kb, ms * 1e3 / 20);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
