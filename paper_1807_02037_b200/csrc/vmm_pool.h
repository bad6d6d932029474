// Device pool over CUDA virtual memory: the budget caps PHYSICAL pages.
//
// The budget's worth of physical pages is created and mapped once,
// contiguously, at the start of a much larger reserved VA range.  Pages are
// 64 MiB (a multiple of the driver's 2 MiB granularity): on B200 the cost of
// cuMemSetAccess / cuMemUnmap is per mapped handle (~0.6 ms / ~0.2 ms for a
// 2 MiB page, measured by scripts/micro/vmm_cost.cu), so large pages make a
// page move ~16x cheaper per byte.  Two best-fit arenas carve the VA: small
// blocks (<= 1 MiB, 512 B granules) and large blocks (2 MiB granules); blocks
// share pages, and a page can move only when no live block touches it.  While the mapped region has a free range that fits, this
// is an ordinary caching allocator: split and merge in place, no driver call.
// Only when fragmentation leaves no mapped range large enough does the pool
// move pages: it unmaps idle pages of free ranges and maps them under a free
// VA range that fits (usually the unmapped tail), so a request that fits the
// budget never fails for lack of contiguity.
//
// A page move does not unmap the page from its old VA: cuMemUnmap waits for
// the device to drain (measured: 10x spread in host time depending on the
// queue), so the page is mapped at the new VA as an alias and the old VA
// page becomes a "zombie" mapping nobody may allocate over.  Zombies are
// unmapped in bulk by trim() at a quiet point (step end, synchronize), or
// individually when their VA is needed again (last resort).
//
// "Idle" is decided without device-wide synchronisation: every free records
// an event on the freeing stream and stamps the block with that stream's
// clock value; a block is idle once its stream's clock has passed the stamp.
//
// Driver entry points come from cudaGetDriverEntryPoint (no link-time libcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <deque>
#include <string>
#include <unordered_map>
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

// Per-stream logical clock: stamp() records an event and returns a number;
// passed(s) says whether all work enqueued before stamp s has finished.
class StreamClocks {
 public:
  ~StreamClocks() {
    for (auto& kv : clocks_)
      for (auto& p : kv.second.pending) cudaEventDestroy(p.second);
    for (auto e : spare_) cudaEventDestroy(e);
  }
  uint64_t stamp(void* stream) {
    Clock& c = clocks_[stream];
    cudaEvent_t e;
    if (!spare_.empty()) {
      e = spare_.back();
      spare_.pop_back();
    } else {
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    cudaEventRecord(e, static_cast<cudaStream_t>(stream));
    uint64_t s = ++c.next;
    c.pending.emplace_back(s, e);
    if (c.pending.size() > 64) poll(c);
    return s;
  }
  bool passed(void* stream, uint64_t s) {
    if (s == 0) return true;
    auto it = clocks_.find(stream);
    if (it == clocks_.end()) return true;
    Clock& c = it->second;
    if (c.done >= s) return true;
    poll(c);
    return c.done >= s;
  }
  // block the host until stamp s on `stream` has passed
  void wait(void* stream, uint64_t s) {
    auto it = clocks_.find(stream);
    if (it == clocks_.end()) return;
    Clock& c = it->second;
    while (c.done < s && !c.pending.empty()) {
      cudaEventSynchronize(c.pending.front().second);
      poll(c);
    }
  }
  // make `waiter` wait (on the device) for stamp s of `stream`
  void device_wait(void* waiter, void* stream, uint64_t s) {
    auto it = clocks_.find(stream);
    if (it == clocks_.end()) return;
    for (auto& p : it->second.pending)
      if (p.first >= s) {
        cudaStreamWaitEvent(static_cast<cudaStream_t>(waiter), p.second, 0);
        return;
      }
  }

 private:
  struct Clock {
    std::deque<std::pair<uint64_t, cudaEvent_t>> pending;
    uint64_t next = 0, done = 0;
  };
  void poll(Clock& c) {
    while (!c.pending.empty() && cudaEventQuery(c.pending.front().second) == cudaSuccess) {
      c.done = c.pending.front().first;
      spare_.push_back(c.pending.front().second);
      c.pending.pop_front();
    }
  }
  std::unordered_map<void*, Clock> clocks_;
  std::vector<cudaEvent_t> spare_;
};

class VmmPool {
 public:
  static constexpr size_t kSmallMax = size_t(1) << 20;

  ~VmmPool() { teardown(); }

  // reserve VA, create `limit_bytes` of pages and map them at the start of
  // the large region
  bool init(int device, size_t limit_bytes, void* fresh, std::string* err, size_t page_bytes = size_t(64) << 20) {
    if (!drv_.load(err)) return false;
    fresh_ = fresh;
    prop_ = CUmemAllocationProp{};
    prop_.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop_.location.id = device;
    size_t g = 0;
    if (drv_.granularity(&g, &prop_, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || g == 0) {
      *err = "cuMemGetAllocationGranularity failed";
      return false;
    }
    gran_ = g;
    page_ = std::max(g, (page_bytes + g - 1) / g * g);
    limit_pages_ = limit_bytes / page_;
    small_va_ = size_t(8) << 30;
    large_va_ = std::max(4 * limit_pages_ * page_, size_t(64) << 30);
    CUdeviceptr base = 0;
    if (drv_.reserve(&base, small_va_ + large_va_, page_, 0, 0) != CUDA_SUCCESS) {
      *err = "cuMemAddressReserve failed";
      return false;
    }
    base_ = reinterpret_cast<char*>(base);
    small_.init(base_, small_va_, fresh, Arena::kAlign);
    large_.init(base_ + small_va_, large_va_, fresh, gran_);
    handle_of_.assign((small_va_ + large_va_) / page_, -1);
    zombie_.assign(handle_of_.size(), -1);
    live_.assign(handle_of_.size(), 0);
    access_.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    access_.location.id = device;
    access_.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    auto t0 = now();
    for (size_t i = 0; i < limit_pages_; ++i) {
      CUmemGenericAllocationHandle hd = 0;
      if (drv_.create(&hd, page_, &prop_, 0) != CUDA_SUCCESS) {
        *err = "cuMemCreate failed (not enough device memory for the budget?)";
        return false;
      }
      handles_.push_back(hd);
      free_.push_back(int(i));
    }
    created_ = limit_pages_;
    driver_s_ += secs(t0);
    // map the whole budget contiguously at the start of the large region
    size_t first = small_va_ / page_;
    std::vector<size_t> pages(limit_pages_);
    for (size_t i = 0; i < limit_pages_; ++i) pages[i] = first + i;
    return map_pages(pages, err);
  }

  size_t page() const { return page_; }
  size_t limit_bytes() const { return limit_pages_ * page_; }
  char* base() const { return base_; }
  bool owns(const void* p) const {
    const char* c = static_cast<const char*>(p);
    return base_ && c >= base_ && c < base_ + small_va_ + large_va_;
  }
  Arena& arena_for(size_t size) { return size <= kSmallMax ? small_ : large_; }
  Arena& arena_of(const void* p) { return static_cast<const char*>(p) < base_ + small_va_ ? small_ : large_; }
  char* ptr(const Block* b) const { return b->owner->base() + b->off; }
  Block* find(const void* p) {
    Arena& a = arena_of(p);
    return a.find_live(static_cast<const char*>(p) - a.base());
  }
  Block* containing(const void* p) {
    Arena& a = arena_of(p);
    return a.containing(static_cast<const char*>(p) - a.base());
  }

  // Allocate `size` bytes for `stream`.  On success the block is live and
  // backed; *wait_stream/*wait_seq name a stamp the caller's stream must
  // device-wait on (cross-stream reuse of a range not yet idle), or null.
  // allow_moves=false: only ranges whose pages are all mapped qualify (no driver call)
  Block* alloc(size_t size, void* stream, bool may_block, std::string* err, bool allow_moves = true) {
    Arena& ar = arena_for(size);
    Block* b = ar.alloc_scored(size, [&](const Block* fb, size_t sz) -> long {
      long unmapped = long(unmapped_in(ar, fb->off, sz));
      long foreign = (fb->tag != stream && fb->tag != fresh_) ? 1 : 0;
      return 4 * unmapped + foreign;
    });
    if (!b) {
      *err = "VA exhausted";
      return nullptr;
    }
    if (!allow_moves && unmapped_in(ar, b->off, b->size) > 0) {
      ar.release(b);
      *err = "no mapped range fits";
      return nullptr;
    }
    pin(b, +1);
    size_t f, l;
    span(b, &f, &l);
    std::vector<size_t> need;
    for (size_t p = f; p <= l; ++p)
      if (handle_of_[p] < 0) need.push_back(p);
    if (!need.empty() && !(steal(need.size(), may_block) && map_pages(need, err))) {
      pin(b, -1);
      ar.release(b);
      if (err->empty()) *err = "physical page budget exhausted (no idle pages to move)";
      return nullptr;
    }
    bytes_live_ += b->size;
    return b;
  }

  void free(Block* b, void* stream, uint64_t seq) {
    bytes_live_ -= b->size;
    pin(b, -1);
    b->tag = stream;
    b->seq = seq;
    b->owner->release(b);
  }

  // cross-stream reuse check for a freshly allocated block (before retagging)
  bool idle(const Block* b) { return b->tag == fresh_ || clocks_.passed(b->tag, b->seq); }

  size_t live_bytes() const { return bytes_live_; }
  size_t live_pages() const { return live_pages_; }
  size_t limit_pages() const { return limit_pages_; }
  size_t mapped_bytes() const { return mapped_ * page_; }
  uint64_t n_map() const { return n_map_; }
  uint64_t n_unmap() const { return n_unmap_; }
  uint64_t n_moves() const { return n_moves_; }
  double driver_ms() const { return driver_s_ * 1e3; }
  size_t zombies() const { return n_zombie_; }
  // unmap every zombie alias (call where a device drain costs nothing)
  void trim() {
    if (!n_zombie_) return;
    for (size_t p = 0; p < zombie_.size() && n_zombie_; ++p)
      if (zombie_[p] >= 0) unmap_zombie(p);
  }
  double unmap_ms() const { return unmap_s_ * 1e3; }
  double map_ms() const { return map_s_ * 1e3; }
  double access_ms() const { return access_s_ * 1e3; }
  size_t va_bytes() const { return small_va_ + large_va_; }
  template <class F>
  void for_each_live(F&& f) {
    small_.for_each_live([&](Block* b) { f(uint64_t(b->size)); });
    large_.for_each_live([&](Block* b) { f(uint64_t(b->size)); });
  }

  StreamClocks clocks_;

 private:
  static std::chrono::steady_clock::time_point now() { return std::chrono::steady_clock::now(); }
  static double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(now() - t0).count();
  }

  void span(const Block* b, size_t* f, size_t* l) const {
    size_t lo = size_t(b->owner->base() - base_) + b->off;
    *f = lo / page_;
    *l = (lo + b->size - 1) / page_;
  }
  size_t unmapped_in(const Arena& a, size_t off, size_t size) const {
    size_t lo = size_t(a.base() - base_) + off;
    size_t f = lo / page_, l = (lo + a.round_up(size) - 1) / page_, n = 0;
    for (size_t p = f; p <= l; ++p) n += handle_of_[p] < 0 ? (zombie_[p] >= 0 ? 8 : 1) : 0;
    return n;
  }
  void pin(const Block* b, int d) {
    size_t f, l;
    span(b, &f, &l);
    for (size_t p = f; p <= l; ++p) {
      uint32_t before = live_[p];
      live_[p] = uint32_t(int(before) + d);
      live_pages_ += (before == 0 && live_[p] > 0) - (before > 0 && live_[p] == 0);
    }
  }

  // make `n` pages free by unmapping idle pages of free ranges (no live
  // block on them, last user finished); optionally wait for busy ones
  bool steal(size_t n, bool may_block) {
    if (free_.size() >= n) return true;
    ++n_moves_;
    for (int pass = 0; pass < 2 && free_.size() < n; ++pass) {
      if (pass == 1 && !may_block) break;
      std::vector<Block*> cands;
      auto collect = [&](Block* fb) { cands.push_back(fb); };
      large_.for_each_free(collect);
      small_.for_each_free(collect);
      // smallest ranges first: they are the fragments nobody can use
      std::sort(cands.begin(), cands.end(), [](const Block* a, const Block* b) { return a->size < b->size; });
      for (Block* fb : cands) {
        if (free_.size() >= n) break;
        if (fb->tag != fresh_ && !clocks_.passed(fb->tag, fb->seq)) {
          if (pass == 0) continue;
          clocks_.wait(fb->tag, fb->seq);
        }
        size_t f, l;
        span(fb, &f, &l);
        // only pages the free range owns entirely and no live block touches
        for (size_t p = l + 1; p-- > f && free_.size() < n;) {
          if (handle_of_[p] >= 0 && live_[p] == 0) retire_page(p);
        }
      }
    }
    return free_.size() >= n;
  }

  // move-out of a page: its physical handle becomes free for another VA while
  // the old mapping stays as a zombie (no cuMemUnmap on the hot path)
  void retire_page(size_t p) {
    free_.push_back(handle_of_[p]);
    zombie_[p] = handle_of_[p];
    handle_of_[p] = -1;
    --mapped_;
    ++n_zombie_;
    ++n_unmap_;
  }

  void unmap_zombie(size_t p) {
    auto t0 = now();
    drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
    const double dt = secs(t0);
    driver_s_ += dt;
    unmap_s_ += dt;
    zombie_[p] = -1;
    --n_zombie_;
  }


  bool map_pages(const std::vector<size_t>& pages, std::string* err) {
    auto t0 = now();
    size_t run = 0;
    for (size_t i = 0; i < pages.size(); ++i) {
      int h = free_.back();
      free_.pop_back();
      size_t p = pages[i];
      if (zombie_[p] >= 0) unmap_zombie(p);   // its VA is needed again
      auto tm = now();
      const CUresult mr = drv_.map(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_, 0, handles_[h], 0);
      map_s_ += secs(tm);
      if (mr != CUDA_SUCCESS) {
        free_.push_back(h);
        *err = "cuMemMap failed";
        driver_s_ += secs(t0);
        return false;
      }
      handle_of_[p] = h;
      ++mapped_;
      ++n_map_;
      bool last = i + 1 == pages.size() || pages[i + 1] != p + 1;
      if (last) {
        size_t start = pages[run];
        auto ta = now();
        const CUresult ar = drv_.set_access(reinterpret_cast<CUdeviceptr>(base_ + start * page_),
                                            (p - start + 1) * page_, &access_, 1);
        access_s_ += secs(ta);
        if (ar != CUDA_SUCCESS) {
          *err = "cuMemSetAccess failed";
          driver_s_ += secs(t0);
          return false;
        }
        run = i + 1;
      }
    }
    driver_s_ += secs(t0);
    return true;
  }

  void teardown() {
    if (!base_) return;
    for (size_t p = 0; p < handle_of_.size(); ++p) {
      if (handle_of_[p] >= 0) drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
      if (zombie_[p] >= 0) drv_.unmap(reinterpret_cast<CUdeviceptr>(base_ + p * page_), page_);
    }
    for (auto h : handles_) drv_.release(h);
    drv_.address_free(reinterpret_cast<CUdeviceptr>(base_), small_va_ + large_va_);
    base_ = nullptr;
  }

  Drv drv_;
  CUmemAllocationProp prop_{};
  CUmemAccessDesc access_{};
  void* fresh_ = nullptr;
  size_t page_ = size_t(64) << 20, gran_ = size_t(2) << 20;
  size_t small_va_ = 0, large_va_ = 0;
  char* base_ = nullptr;
  Arena small_, large_;
  std::vector<int32_t> handle_of_;   // VA page -> physical page (-1: unmapped)
  std::vector<int32_t> zombie_;      // VA page -> stale alias of a moved page (-1: none)
  size_t n_zombie_ = 0;
  std::vector<uint32_t> live_;       // VA page -> live blocks touching it
  std::vector<CUmemGenericAllocationHandle> handles_;
  std::vector<int> free_;            // physical pages not mapped anywhere
  size_t created_ = 0, limit_pages_ = 0, mapped_ = 0, bytes_live_ = 0, live_pages_ = 0;
  uint64_t n_map_ = 0, n_unmap_ = 0, n_moves_ = 0;
  double driver_s_ = 0, unmap_s_ = 0, map_s_ = 0, access_s_ = 0;
};

}  // namespace lms
