// Device pool over CUDA virtual memory: the budget caps PHYSICAL pages.
//
// Physical memory is a fixed set of pages (the driver's allocation
// granularity, 2 MiB on B200) created once, up front, up to the budget.
// Virtual address space is reserved generously and never limits anything.
//
// * Large blocks (> 1 MiB) get their own page-aligned VA range with pages
//   mapped in.  A freed large block stays mapped in an exact-size cache with
//   the event recorded at free: a training step allocates the same multiset
//   of sizes every iteration, so steady-state allocation is a cache hit with
//   no driver call.  When an allocation needs pages and none are free, the
//   least recently freed cached block whose event has completed is unmapped
//   (its VA range goes back to the VA arena, its pages to the free list); no
//   device-wide synchronisation is needed because each cached block knows
//   when its last user finished.
// * Small blocks (<= 1 MiB) are sub-allocated from a dedicated VA region
//   whose pages are mapped on first use and stay mapped.
//
// A hole in VA therefore never wastes HBM, and a step fits the budget iff its
// live bytes (rounded to pages) do: fragmentation cannot cause an OOM.
//
// Driver entry points come from cudaGetDriverEntryPoint (no link-time libcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <list>
#include <map>
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

// one large block: a VA range (owned by the VA arena) with `pages` mapped
struct Big {
  Block* va = nullptr;      // range in the VA arena
  size_t pages = 0;
  size_t bytes = 0;         // requested size rounded to 512 B
  void* stream = nullptr;   // last user
  cudaEvent_t ev = nullptr; // recorded when freed; completes when the last user is done
  std::list<Big*>::iterator lru;
  std::vector<int> handles; // physical page per VA page
};

class VmmPool {
 public:
  static constexpr size_t kSmallMax = size_t(1) << 20;

  ~VmmPool() { teardown(); }

  bool init(int device, size_t limit_bytes, size_t va_bytes, void* fresh, std::string* err) {
    if (!drv_.load(err)) return false;
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
    large_va_ = std::max(va_bytes, size_t(64) << 30);
    large_va_ = (large_va_ + page_ - 1) / page_ * page_;
    CUdeviceptr base = 0;
    if (drv_.reserve(&base, small_va_ + large_va_, page_, 0, 0) != CUDA_SUCCESS) {
      *err = "cuMemAddressReserve failed";
      return false;
    }
    base_ = reinterpret_cast<char*>(base);
    small_.init(base_, small_va_, fresh, Arena::kAlign);
    va_.init(base_ + small_va_, large_va_, nullptr, page_);
    small_pages_.assign(small_va_ / page_, -1);
    small_live_.assign(small_va_ / page_, 0);
    access_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    access_.location.id = device;
    access_.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    set_limit(limit_bytes);
    return true;
  }

  // create physical pages up front (cuMemCreate is the slow driver call)
  bool precreate(size_t pages, std::string* err) {
    auto t0 = now();
    while (created_ < std::min(pages, limit_pages_)) {
      CUmemGenericAllocationHandle hd = 0;
      if (drv_.create(&hd, page_, &prop_, 0) != CUDA_SUCCESS) {
        *err = "cuMemCreate failed while pre-creating pages";
        driver_s_ += secs(t0);
        return false;
      }
      handles_.push_back(hd);
      free_.push_back(int(handles_.size()) - 1);
      ++created_;
    }
    driver_s_ += secs(t0);
    return true;
  }

  void set_limit(size_t bytes) { limit_pages_ = bytes / page_; }
  size_t limit_bytes() const { return limit_pages_ * page_; }
  size_t page() const { return page_; }
  char* base() const { return base_; }
  bool owns(const void* p) const {
    const char* c = static_cast<const char*>(p);
    return base_ && c >= base_ && c < base_ + small_va_ + large_va_;
  }
  bool is_small(const void* p) const { return static_cast<const char*>(p) < base_ + small_va_; }

  // ---- small blocks -------------------------------------------------------
  // nullptr when pages are short (the caller evicts or waits and retries)
  Block* small_alloc(size_t size, void* stream, std::string* err) {
    Block* b = small_.alloc(size, stream);
    if (!b) {
      *err = "small-block VA exhausted";
      return nullptr;
    }
    size_t f = b->off / page_, l = (b->off + b->size - 1) / page_;
    size_t need = 0;
    for (size_t p = f; p <= l; ++p) need += small_pages_[p] < 0;
    if (need > spare_pages()) {
      small_.release(b);
      *err = "physical page budget exhausted";
      return nullptr;
    }
    for (size_t p = f; p <= l; ++p) {
      if (small_pages_[p] < 0) {
        int h = take_page();
        if (!map_pages(base_ + p * page_, &h, 1, err)) {
          give_page(h);
          for (size_t q = f; q < p; ++q) --small_live_[q];
          small_.release(b);
          return nullptr;
        }
        small_pages_[p] = h;
        ++small_mapped_;
      }
      ++small_live_[p];
    }
    small_bytes_ += b->size;
    return b;
  }
  void small_free(Block* b) {
    size_t f = b->off / page_, l = (b->off + b->size - 1) / page_;
    for (size_t p = f; p <= l; ++p) --small_live_[p];
    small_bytes_ -= b->size;
    small_.release(b);
  }
  Block* small_find(const void* p) { return small_.find_live(static_cast<const char*>(p) - base_); }
  Block* small_containing(const void* p) { return small_.containing(static_cast<const char*>(p) - base_); }
  char* small_ptr(const Block* b) const { return base_ + b->off; }
  Arena& small_arena() { return small_; }

  // ---- large blocks --------------------------------------------------------
  // exact-size cache hit: the caller's stream first (stream order makes the
  // reuse safe), then a block whose last user finished, then any (the caller
  // must make its stream wait on the returned block's event)
  Big* big_from_cache(size_t pages, void* stream, bool* needs_wait) {
    auto range = cache_.equal_range(pages);
    auto done = cache_.end(), any = cache_.end();
    for (auto it = range.first; it != range.second; ++it) {
      Big* b = it->second;
      if (b->stream == stream) return take_cached(it, needs_wait, false);
      if (done == cache_.end() && (b->ev == nullptr || cudaEventQuery(b->ev) == cudaSuccess)) done = it;
      if (any == cache_.end()) any = it;
    }
    if (done != cache_.end()) return take_cached(done, needs_wait, false);
    if (any != cache_.end()) return take_cached(any, needs_wait, true);
    return nullptr;
  }

  // fresh VA + pages, evicting finished cached blocks for pages (waiting for
  // unfinished ones only if `wait_for_cache`).  nullptr if the budget cannot
  // supply `pages`.
  Big* big_fresh(size_t bytes, size_t pages, bool wait_for_cache, std::string* err) {
    while (spare_pages() < pages) {
      if (!evict_one(wait_for_cache)) {
        *err = "physical page budget exhausted";
        return nullptr;
      }
    }
    Block* va = va_.alloc(pages * page_);
    if (!va) {
      *err = "large-block VA exhausted";
      return nullptr;
    }
    Big* b = new Big();
    b->va = va;
    b->pages = pages;
    b->bytes = bytes;
    b->handles.resize(pages);
    for (size_t i = 0; i < pages; ++i) b->handles[i] = take_page();
    if (!map_pages(va_.base() + va->off, b->handles.data(), pages, err)) {
      for (int h : b->handles) give_page(h);
      va_.release(va);
      delete b;
      return nullptr;
    }
    big_mapped_ += pages;
    return b;
  }

  void big_live(Big* b, size_t bytes) {
    b->bytes = bytes;
    live_[ptr(b)] = b;
    big_live_pages_ += b->pages;
    big_bytes_ += b->bytes;
  }

  // freed by `stream`: cache it, with `ev` marking its last use
  void big_free(Big* b, void* stream, cudaEvent_t ev) {
    live_.erase(ptr(b));
    big_live_pages_ -= b->pages;
    big_bytes_ -= b->bytes;
    b->stream = stream;
    b->ev = ev;
    lru_.push_back(b);
    b->lru = std::prev(lru_.end());
    cache_.emplace(b->pages, b);
  }

  Big* big_find(const void* p) {
    auto it = live_.find(const_cast<char*>(static_cast<const char*>(p)));
    return it == live_.end() ? nullptr : it->second;
  }
  Big* big_containing(const void* p) {
    char* c = const_cast<char*>(static_cast<const char*>(p));
    auto it = live_.upper_bound(c);
    if (it == live_.begin()) return nullptr;
    --it;
    return c < it->first + it->second->pages * page_ ? it->second : nullptr;
  }
  char* ptr(const Big* b) const { return va_.base() + b->va->off; }

  // evict cached blocks until `pages` pages are spare
  bool make_room(size_t pages, bool wait) {
    while (spare_pages() < pages)
      if (!evict_one(wait)) return false;
    return true;
  }

  // unmap every cached block (only when no cached block can be in use)
  void flush_cache() {
    while (!lru_.empty()) evict(lru_.front());
  }
  bool has_cache() const { return !lru_.empty(); }

  // ---- accounting ------------------------------------------------------------
  size_t mapped_pages() const { return small_mapped_ + big_mapped_; }
  size_t spare_pages() const {
    size_t m = mapped_pages();
    if (m >= limit_pages_) return 0;
    size_t creatable = created_ < limit_pages_ ? limit_pages_ - created_ : 0;
    return std::min(limit_pages_ - m, free_.size() + creatable);
  }
  size_t live_pages() const { return big_live_pages_ + (small_bytes_ + page_ - 1) / page_; }
  size_t live_bytes() const { return big_bytes_ + small_bytes_; }
  size_t mapped_bytes() const { return mapped_pages() * page_; }
  size_t cached_bytes() const { return (big_mapped_ - big_live_pages_) * page_; }
  uint64_t n_map() const { return n_map_; }
  uint64_t n_unmap() const { return n_unmap_; }
  uint64_t n_hits() const { return n_hits_; }
  double driver_ms() const { return driver_s_ * 1e3; }
  size_t va_bytes() const { return small_va_ + large_va_; }
  size_t largest_free_va() const { return va_.largest_free(); }
  template <class F>
  void for_each_live(F&& f) {
    small_.for_each_live([&](Block* b) { f(uint64_t(b->size)); });
    for (auto& kv : live_) f(uint64_t(kv.second->bytes));
  }

  // events of evicted blocks, handed back to the owner's event pool
  std::vector<cudaEvent_t> events_done_;

 private:
  static std::chrono::steady_clock::time_point now() { return std::chrono::steady_clock::now(); }
  static double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(now() - t0).count();
  }

  Big* take_cached(std::multimap<size_t, Big*>::iterator it, bool* needs_wait, bool wait) {
    Big* b = it->second;
    cache_.erase(it);
    lru_.erase(b->lru);
    *needs_wait = wait;
    ++n_hits_;
    return b;
  }

  int take_page() {
    if (!free_.empty()) {
      int h = free_.back();
      free_.pop_back();
      return h;
    }
    CUmemGenericAllocationHandle hd = 0;
    if (created_ >= limit_pages_ || drv_.create(&hd, page_, &prop_, 0) != CUDA_SUCCESS) return -1;
    handles_.push_back(hd);
    ++created_;
    return int(handles_.size()) - 1;
  }
  void give_page(int h) {
    if (h >= 0) free_.push_back(h);
  }

  bool map_pages(char* va, const int* hs, size_t n, std::string* err) {
    auto t0 = now();
    for (size_t i = 0; i < n; ++i) {
      if (hs[i] < 0 || drv_.map(reinterpret_cast<CUdeviceptr>(va + i * page_), page_, 0, handles_[hs[i]], 0) !=
                           CUDA_SUCCESS) {
        for (size_t j = 0; j < i; ++j) drv_.unmap(reinterpret_cast<CUdeviceptr>(va + j * page_), page_);
        *err = "cuMemMap failed";
        driver_s_ += secs(t0);
        return false;
      }
    }
    n_map_ += n;
    bool ok = drv_.set_access(reinterpret_cast<CUdeviceptr>(va), n * page_, &access_, 1) == CUDA_SUCCESS;
    if (!ok) *err = "cuMemSetAccess failed";
    driver_s_ += secs(t0);
    return ok;
  }

  void evict(Big* b) {
    auto t0 = now();
    char* va = ptr(b);
    for (size_t i = 0; i < b->pages; ++i) drv_.unmap(reinterpret_cast<CUdeviceptr>(va + i * page_), page_);
    driver_s_ += secs(t0);
    n_unmap_ += b->pages;
    for (int h : b->handles) give_page(h);
    big_mapped_ -= b->pages;
    auto range = cache_.equal_range(b->pages);
    for (auto it = range.first; it != range.second; ++it)
      if (it->second == b) {
        cache_.erase(it);
        break;
      }
    lru_.erase(b->lru);
    va_.release(b->va);
    if (b->ev) events_done_.push_back(b->ev);
    delete b;
  }

  // evict the least recently freed cached block whose last user finished
  // (or, if `wait`, the oldest one after waiting for it)
  bool evict_one(bool wait) {
    for (Big* b : lru_) {
      if (b->ev == nullptr || cudaEventQuery(b->ev) == cudaSuccess) {
        evict(b);
        return true;
      }
    }
    if (wait && !lru_.empty()) {
      Big* b = lru_.front();
      if (b->ev) cudaEventSynchronize(b->ev);
      evict(b);
      return true;
    }
    return false;
  }

  void teardown() {
    if (!base_) return;
    while (!lru_.empty()) evict(lru_.front());
    for (auto& kv : live_) {
      for (size_t i = 0; i < kv.second->pages; ++i)
        drv_.unmap(reinterpret_cast<CUdeviceptr>(kv.first + i * page_), page_);
      delete kv.second;
    }
    for (size_t p = 0; p < small_pages_.size(); ++p)
      if (small_pages_[p] >= 0) drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
    for (auto h : handles_)
      if (h) drv_.release(h);
    drv_.address_free(reinterpret_cast<CUdeviceptr>(base_), small_va_ + large_va_);
    base_ = nullptr;
  }

  Drv drv_;
  CUmemAllocationProp prop_{};
  CUmemAccessDesc access_{};
  size_t page_ = size_t(2) << 20;
  size_t small_va_ = 0, large_va_ = 0;
  char* base_ = nullptr;

  Arena small_;                          // small blocks over the first region
  std::vector<int32_t> small_pages_;     // small-region page -> handle (-1 unmapped)
  std::vector<uint32_t> small_live_;     // small-region page -> live blocks
  size_t small_mapped_ = 0, small_bytes_ = 0;

  Arena va_;                             // unmapped VA of the large region
  std::map<char*, Big*> live_;           // live large blocks by address
  std::multimap<size_t, Big*> cache_;    // pages -> cached (free, mapped) block
  std::list<Big*> lru_;                  // cached blocks, least recently freed first
  size_t big_mapped_ = 0, big_live_pages_ = 0, big_bytes_ = 0;

  std::vector<CUmemGenericAllocationHandle> handles_;
  std::vector<int> free_;                // created, unmapped pages
  size_t created_ = 0, limit_pages_ = 0;
  uint64_t n_map_ = 0, n_unmap_ = 0, n_hits_ = 0;
  double driver_s_ = 0;
};

}  // namespace lms
