// Driver-call costs of the VMM operations the device pool uses (B200).
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  cudaFree(0);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED; prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = 0;
  size_t g = 0; cuMemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  CUmemAccessDesc acc{}; acc.location = prop.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t mult : {1, 16}) {
    size_t pg = g * mult; int N = int(2048 / mult);  // 4 GiB worth
    std::vector<CUmemGenericAllocationHandle> h(N);
    double t = now(); for (int i = 0; i < N; ++i) cuMemCreate(&h[i], pg, &prop, 0); double tc = now() - t;
    CUdeviceptr va; cuMemAddressReserve(&va, N * pg * 2, pg, 0, 0);
    t = now(); for (int i = 0; i < N; ++i) cuMemMap(va + i * pg, pg, 0, h[i], 0); double tm = now() - t;
    t = now(); cuMemSetAccess(va, N * pg, &acc, 1); double ta1 = now() - t;
    t = now(); for (int i = 0; i < N; ++i) cuMemUnmap(va + i * pg, pg); double tu = now() - t;
    t = now(); for (int i = 0; i < N; ++i) cuMemMap(va + i * pg, pg, 0, h[i], 0); double tm2 = now() - t;
    t = now(); for (int i = 0; i < N; ++i) cuMemSetAccess(va + i * pg, pg, &acc, 1); double taN = now() - t;
    // remap half the pages to the second half of the VA (a "move"), with kernels idle
    t = now();
    for (int i = 0; i < N / 2; ++i) { cuMemUnmap(va + i * pg, pg); cuMemMap(va + (N + i) * pg, pg, 0, h[i], 0); }
    cuMemSetAccess(va + N * pg, (N / 2) * pg, &acc, 1);
    double tmove = now() - t;
    printf("page %zu MiB x %d: create %.1f us/page, map %.1f/%.1f us/page, set_access one-range %.1f ms, "
           "per-page %.1f us, unmap %.1f us/page, move %.1f us/page\n",
           pg >> 20, N, tc / N * 1e6, tm / N * 1e6, tm2 / N * 1e6, ta1 * 1e3, taN / N * 1e6, tu / N * 1e6,
           tmove / (N / 2) * 1e6);
  }
  return 0;
}
