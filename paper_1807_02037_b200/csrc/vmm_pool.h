// Device pool over CUDA virtual memory: the budget caps PHYSICAL pages.
//
// Virtual address space is reserved generously (several times the budget)
// and carved by two best-fit arenas: a small-block arena (512 B granules,
// blocks <= 1 MiB, several blocks per page) and a large-block arena
// (page-aligned).  Physical memory comes in fixed pages (the driver's
// allocation granularity, 2 MiB on B200) mapped into a block's VA range on
// demand.  Freed blocks keep their pages mapped (a cache: reusing a range
// costs no driver call); when an allocation needs more pages than the budget
// leaves, pages of free ranges are unmapped and remapped where needed.  So a
// hole in VA never wastes HBM, and "does the step fit the budget" means
// exactly "are the live bytes (rounded to pages) under the budget" — the
// fragmentation that sinks a contiguous arena cannot cause an OOM here.
//
// Driver entry points are fetched with cudaGetDriverEntryPoint, so the
// library needs no link-time libcuda.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <string>
#include <vector>

#include "arena.h"

namespace lms {

struct Drv {
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) address_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;

  bool load(std::string* err) {
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
      if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || *fn == nullptr) {
        *err = std::string("driver entry point missing: ") + name;
        return false;
      }
      return true;
    };
    return get("cuMemAddressReserve", (void**)&reserve) && get("cuMemAddressFree", (void**)&address_free) &&
           get("cuMemCreate", (void**)&create) && get("cuMemRelease", (void**)&release) &&
           get("cuMemMap", (void**)&map) && get("cuMemUnmap", (void**)&unmap) &&
           get("cuMemSetAccess", (void**)&set_access) &&
           get("cuMemGetAllocationGranularity", (void**)&granularity);
  }
};

class VmmPool {
 public:
  static constexpr size_t kSmallMax = size_t(1) << 20;

  ~VmmPool() { teardown(); }

  // reserve VA and set the physical budget; pages are created lazily
  bool init(int device, size_t limit_bytes, size_t va_hint, void* fresh, std::string* err) {
    if (!drv_.load(err)) return false;
    device_ = device;
    prop_ = CUmemAllocationProp{};
    prop_.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop_.location.id = device;
    size_t g = 0;
    if (drv_.granularity(&g, &prop_, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || g == 0) {
      *err = "cuMemGetAllocationGranularity failed";
      return false;
    }
    page_ = g;
    small_va_ = size_t(8) << 30;
    large_va_ = std::max(va_hint, size_t(64) << 30);
    large_va_ = (large_va_ + page_ - 1) / page_ * page_;
    CUdeviceptr base = 0;
    if (drv_.reserve(&base, small_va_ + large_va_, page_, 0, 0) != CUDA_SUCCESS) {
      *err = "cuMemAddressReserve failed";
      return false;
    }
    base_ = reinterpret_cast<char*>(base);
    small_.init(base_, small_va_, fresh, Arena::kAlign);
    large_.init(base_ + small_va_, large_va_, fresh, page_);
    size_t npages = (small_va_ + large_va_) / page_;
    handle_of_.assign(npages, -1);
    live_.assign(npages, 0);
    set_limit(limit_bytes);
    access_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    access_.location.id = device;
    access_.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    return true;
  }

  void set_limit(size_t bytes) { limit_pages_ = bytes / page_; }
  size_t limit_bytes() const { return limit_pages_ * page_; }
  size_t page() const { return page_; }
  bool owns(const void* p) const {
    const char* c = static_cast<const char*>(p);
    return base_ && c >= base_ && c < base_ + small_va_ + large_va_;
  }
  char* base() const { return base_; }

  Arena& arena_for(size_t size) { return size <= kSmallMax ? small_ : large_; }
  Arena& arena_of(const void* p) {
    return static_cast<const char*>(p) < base_ + small_va_ ? small_ : large_;
  }
  char* ptr_of(Arena& a, const Block* b) const { return a.base() + b->off; }

  Block* find_live(const void* p) {
    Arena& a = arena_of(p);
    return a.find_live(static_cast<const char*>(p) - a.base());
  }
  Block* containing(const void* p) {
    Arena& a = arena_of(p);
    return a.containing(static_cast<const char*>(p) - a.base());
  }

  // pages [first, last] touched by block b of arena a
  void page_span(Arena& a, const Block* b, size_t* first, size_t* last) const {
    size_t lo = size_t(a.base() - base_) + b->off;
    *first = lo / page_;
    *last = (lo + b->size - 1) / page_;
  }

  // pages of b that still need physical backing
  size_t unmapped_pages(Arena& a, const Block* b) const {
    size_t f, l, n = 0;
    page_span(a, b, &f, &l);
    for (size_t p = f; p <= l; ++p) n += handle_of_[p] < 0;
    return n;
  }

  // pages that may still be mapped under the budget
  size_t spare_pages() const { return mapped_ >= limit_pages_ ? 0 : limit_pages_ - mapped_; }

  // unmapped pages in the first `size` bytes of free block b (the part an
  // allocation of `size` would use)
  long unmapped_prefix(const Arena& a, const Block* b, size_t size) const {
    size_t lo = size_t(a.base() - base_) + b->off;
    size_t f = lo / page_, l = (lo + size - 1) / page_;
    long n = 0;
    for (size_t p = f; p <= l; ++p) n += handle_of_[p] < 0;
    return n;
  }

  void pin(Arena& a, const Block* b, int delta) {
    size_t f, l;
    page_span(a, b, &f, &l);
    for (size_t p = f; p <= l; ++p) live_[p] = uint16_t(int(live_[p]) + delta);
  }

  // unmap pages no live block touches until `want` spare pages exist;
  // the caller has made sure no in-flight work uses free ranges.  Pages are
  // taken from the top of the address space down (the large arena grows
  // upward from fresh VA, so the highest cached pages are the coldest).
  size_t reclaim(size_t want) {
    auto t0 = std::chrono::steady_clock::now();
    size_t got = 0;
    for (size_t q = handle_of_.size(); q-- > 0 && spare_pages() < want;) {
      size_t p = q;
      if (handle_of_[p] >= 0 && live_[p] == 0) {
        drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
        free_handles_.push_back(handle_of_[p]);
        handle_of_[p] = -1;
        --mapped_;
        ++got;
        ++n_unmap_;
      }
    }
    // over the (possibly lowered) limit: drop surplus physical pages
    while (created_ > limit_pages_ && !free_handles_.empty()) {
      int h = free_handles_.back();
      drv_.release(handles_[h]);
      handles_[h] = 0;
      free_slots_.push_back(h);
      free_handles_.pop_back();
      --created_;
    }
    driver_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return got;
  }

  // back every page of b with physical memory; false if the budget is short
  bool map_block(Arena& a, const Block* b, std::string* err) {
    size_t f, l;
    page_span(a, b, &f, &l);
    if (unmapped_pages(a, b) == 0) return true;
    auto t0 = std::chrono::steady_clock::now();
    struct Acc {
      double* s;
      std::chrono::steady_clock::time_point t0;
      ~Acc() { *s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    } acc{&driver_s_, t0};
    size_t run = SIZE_MAX;
    for (size_t p = f; p <= l + 1; ++p) {
      bool need = p <= l && handle_of_[p] < 0;
      if (need) {
        int h = take_handle(err);
        if (h < 0) return false;
        CUdeviceptr va = reinterpret_cast<CUdeviceptr>(base_ + p * page_);
        if (drv_.map(va, page_, 0, handles_[h], 0) != CUDA_SUCCESS) {
          free_handles_.push_back(h);
          *err = "cuMemMap failed";
          return false;
        }
        handle_of_[p] = h;
        ++mapped_;
        ++n_map_;
        if (run == SIZE_MAX) run = p;
      }
      if (!need && run != SIZE_MAX) {
        CUdeviceptr va = reinterpret_cast<CUdeviceptr>(base_ + run * page_);
        if (drv_.set_access(va, (p - run) * page_, &access_, 1) != CUDA_SUCCESS) {
          *err = "cuMemSetAccess failed";
          return false;
        }
        run = SIZE_MAX;
      }
    }
    mapped_peak_ = std::max(mapped_peak_, mapped_);
    return true;
  }

  size_t mapped_bytes() const { return mapped_ * page_; }
  size_t created_pages() const { return created_; }
  size_t mapped_peak_bytes() const { return mapped_peak_ * page_; }
  void reset_mapped_peak() { mapped_peak_ = mapped_; }
  uint64_t n_map() const { return n_map_; }
  double driver_ms() const { return driver_s_ * 1e3; }
  uint64_t n_unmap() const { return n_unmap_; }
  size_t va_bytes() const { return small_va_ + large_va_; }

  Arena small_, large_;

 private:
  int take_handle(std::string* err) {
    if (mapped_ >= limit_pages_) {
      *err = "physical page budget exhausted";
      return -1;
    }
    if (!free_handles_.empty()) {
      int h = free_handles_.back();
      free_handles_.pop_back();
      return h;
    }
    CUmemGenericAllocationHandle hd = 0;
    if (drv_.create(&hd, page_, &prop_, 0) != CUDA_SUCCESS) {
      *err = "cuMemCreate failed (device out of physical memory?)";
      return -1;
    }
    int idx;
    if (!free_slots_.empty()) {
      idx = free_slots_.back();
      free_slots_.pop_back();
      handles_[idx] = hd;
    } else {
      idx = int(handles_.size());
      handles_.push_back(hd);
    }
    ++created_;
    return idx;
  }

 public:
  // create physical pages up front (cuMemCreate is the slow driver call) so
  // that steady-state remaps only pay cuMemMap/cuMemSetAccess
  bool precreate(size_t pages, std::string* err) {
    auto t0 = std::chrono::steady_clock::now();
    while (created_ < std::min(pages, limit_pages_)) {
      CUmemGenericAllocationHandle hd = 0;
      if (drv_.create(&hd, page_, &prop_, 0) != CUDA_SUCCESS) {
        *err = "cuMemCreate failed while pre-creating pages";
        return false;
      }
      handles_.push_back(hd);
      free_handles_.push_back(int(handles_.size()) - 1);
      ++created_;
    }
    driver_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
  }

 private:

  void teardown() {
    if (!base_) return;
    for (size_t p = 0; p < handle_of_.size(); ++p)
      if (handle_of_[p] >= 0) drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
    for (auto h : handles_)
      if (h) drv_.release(h);
    drv_.address_free(reinterpret_cast<CUdeviceptr>(base_), small_va_ + large_va_);
    base_ = nullptr;
  }

  Drv drv_;
  int device_ = 0;
  CUmemAllocationProp prop_{};
  CUmemAccessDesc access_{};
  size_t page_ = size_t(2) << 20;
  size_t small_va_ = 0, large_va_ = 0;
  char* base_ = nullptr;
  std::vector<int32_t> handle_of_;      // page -> physical handle index, -1 unmapped
  std::vector<uint16_t> live_;          // page -> live blocks touching it
  std::vector<CUmemGenericAllocationHandle> handles_;
  std::vector<int> free_handles_;       // created, currently unmapped
  std::vector<int> free_slots_;         // released slots in handles_
  size_t created_ = 0, limit_pages_ = 0, mapped_ = 0, mapped_peak_ = 0;
  uint64_t n_map_ = 0, n_unmap_ = 0;
  double driver_s_ = 0;
};

}  // namespace lms
