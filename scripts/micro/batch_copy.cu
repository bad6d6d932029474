// Can the copy engine move a ZVC v3 stream's variable-size tile chunks (fixed
// 16 KiB slots, 8-16 KiB used) at link rate?  cudaMemcpyBatchAsync with one
// copy per tile vs one contiguous copy of the same bytes, H2D and D2H.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a batch_copy.cu -o batch_copy
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

int main() {
  const size_t ntiles = 16384, slot = 16384;
  const size_t total = ntiles * slot;
  char *h, *d;
  cudaHostAlloc(&h, total, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaMalloc(&d, total);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t used : {slot, size_t(14336), size_t(8192)}) {
    std::vector<void*> dst(ntiles), src(ntiles);
    std::vector<size_t> sz(ntiles, used);
    for (int dir = 0; dir < 2; ++dir) {
      for (size_t t = 0; t < ntiles; ++t) {
        dst[t] = dir == 0 ? (void*)(d + t * slot) : (void*)(h + t * slot);
        src[t] = dir == 0 ? (void*)(h + t * slot) : (void*)(d + t * slot);
      }
      cudaMemcpyAttributes attr{};
      attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
      size_t idx = 0, fail = 0;
      float best_batch = 1e9, best_one = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a, s);
        cudaError_t e = cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), ntiles, &attr, &idx, 1, &fail, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("batch error %s\n", cudaGetErrorString(e)); return 1; }
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it) best_batch = ms < best_batch ? ms : best_batch;
        cudaEventRecord(a, s);
        cudaMemcpyAsync(dir == 0 ? d : h, dir == 0 ? h : d, used * ntiles,
                        dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (it) best_one = ms < best_one ? ms : best_one;
      }
      double bytes = double(used) * ntiles;
      printf("%s used %zu B/tile: batch of %zu copies %.2f GB/s, one copy %.2f GB/s\n", dir == 0 ? "H2D" : "D2H",
             used, ntiles, bytes / best_batch / 1e6, bytes / best_one / 1e6);
    }
  }
  return 0;
}
