// Best-fit sub-allocator over one contiguous address range.
//
// Used for the device arena (HBM budget) and for each pinned host chunk.
// Blocks are kept in address order (doubly linked) for O(1) coalescing and
// in a size-ordered set for best-fit lookup.  No CUDA here: stream and
// event semantics live in the pools that own an Arena.
#pragma once

#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <iterator>
#include <map>
#include <set>
#include <utility>
#include <vector>

namespace lms {

struct Block {
  size_t off = 0;
  size_t size = 0;
  bool free = true;
  Block* prev = nullptr;
  Block* next = nullptr;
  void* tag = nullptr;  // owner-defined (last-use stream for device blocks)
  class Arena* owner = nullptr;
  uint64_t seq = 0;     // owner-defined: stream clock value when the block was freed
};

class Arena {
 public:
  static constexpr size_t kAlign = 512;  // default granularity

  Arena() = default;
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  ~Arena() { clear(); }

  // `fresh` tags never-used space: it merges with any neighbour and adopts
  // the neighbour's tag, since it has no pending work on any stream.
  void init(char* base, size_t capacity, void* fresh = nullptr, size_t align = kAlign) {
    clear();
    align_ = align;
    fresh_ = fresh;
    base_ = base;
    cap_ = capacity - capacity % align_;
    if (cap_ == 0) return;
    Block* b = new Block();
    b->off = 0;
    b->size = cap_;
    b->tag = fresh_;
    b->owner = this;
    head_ = b;
    free_.insert({b->size, b});
  }

  static size_t round(size_t n) { return n == 0 ? kAlign : (n + kAlign - 1) / kAlign * kAlign; }
  size_t round_up(size_t n) const { return n == 0 ? align_ : (n + align_ - 1) / align_ * align_; }
  size_t align() const { return align_; }

  // Best fit with a `tag` preference: among free blocks of the smallest
  // adequate size class, the first whose tag matches wins, else the smallest.
  Block* alloc(size_t size, void* tag_pref = nullptr, bool require_tag = false) {
    size = round_up(size);
    auto it = free_.lower_bound({size, nullptr});
    Block* pick = nullptr;
    if (tag_pref != nullptr || require_tag) {
      int scanned = 0;
      for (auto jt = it; jt != free_.end() && scanned < 32; ++jt, ++scanned) {
        if (jt->second->tag == tag_pref) { pick = jt->second; it = jt; break; }
      }
      if (pick == nullptr && require_tag) return nullptr;
    }
    if (pick == nullptr) {
      if (it == free_.end()) return nullptr;
      pick = it->second;
    }
    return take(it, size);
  }

  template <class It>
  Block* take(It it, size_t size) {
    Block* pick = it->second;
    free_.erase(it);
    if (pick->size - size >= align_) {
      Block* rest = new Block();
      rest->off = pick->off + size;
      rest->size = pick->size - size;
      rest->tag = pick->tag;
      rest->seq = pick->seq;
      rest->owner = this;
      rest->prev = pick;
      rest->next = pick->next;
      if (pick->next) pick->next->prev = rest;
      pick->next = rest;
      pick->size = size;
      free_.insert({rest->size, rest});
    }
    pick->free = false;
    pick->owner = this;
    used_ += pick->size;
    if (used_ > peak_) peak_ = used_;
    live_[pick->off] = pick;
    return pick;
  }

  Block* find_live(size_t off) const {
    auto it = live_.find(off);
    return it == live_.end() ? nullptr : it->second;
  }

  // Return a block; merges with free neighbours that carry the same tag.
  void release(Block* b) {
    live_.erase(b->off);
    used_ -= b->size;
    b->free = true;
    if (b->prev && b->prev->free && mergeable(b->prev, b)) {
      Block* p = b->prev;
      free_.erase({p->size, p});
      if (p->tag == fresh_) p->tag = b->tag;
      // same stream (or fresh): the later free stamp covers both
      p->seq = std::max(p->seq, b->seq);
      p->size += b->size;
      p->next = b->next;
      if (b->next) b->next->prev = p;
      delete b;
      b = p;
    }
    if (b->next && b->next->free && mergeable(b, b->next)) {
      Block* n = b->next;
      free_.erase({n->size, n});
      if (b->tag == fresh_) b->tag = n->tag;
      b->seq = std::max(b->seq, n->seq);
      b->size += n->size;
      b->next = n->next;
      if (n->next) n->next->prev = b;
      delete n;
    }
    free_.insert({b->size, b});
  }

  // Give every free block `tag` and coalesce runs of adjacent free blocks
  // (used once nothing is pending on any stream, e.g. after a device sync).
  void retag_all_free(void* tag) {
    free_.clear();
    Block* b = head_;
    while (b) {
      if (b->free) {
        b->tag = tag;
        while (b->next && b->next->free) {
          Block* n = b->next;
          b->size += n->size;
          b->next = n->next;
          if (n->next) n->next->prev = b;
          delete n;
        }
        free_.insert({b->size, b});
      }
      b = b->next;
    }
  }

  bool mergeable(const Block* a, const Block* b) const {
    return a->tag == b->tag || a->tag == fresh_ || b->tag == fresh_;
  }

  // Best fit guided by a cost: among the first `scan` free blocks of adequate
  // size (ascending size), take the lowest cost(block, size); ties keep the
  // smaller block.  Lets the device pool prefer ranges whose pages are mapped.
  template <class Cost>
  Block* alloc_scored(size_t size, Cost cost, int scan = 48) {
    size = round_up(size);
    auto it = free_.lower_bound({size, nullptr});
    if (it == free_.end()) return nullptr;
    auto best = it;
    long best_cost = cost(it->second, size);
    int n = 1;
    for (auto jt = std::next(it); jt != free_.end() && n < scan && best_cost > 0; ++jt, ++n) {
      long c = cost(jt->second, size);
      if (c < best_cost) {
        best_cost = c;
        best = jt;
      }
    }
    return take(best, size);
  }

  // Live block containing the byte at `off`, or nullptr.
  Block* containing(size_t off) const {
    auto it = live_.upper_bound(off);
    if (it == live_.begin()) return nullptr;
    --it;
    Block* b = it->second;
    return (off < b->off + b->size) ? b : nullptr;
  }

  size_t largest_free() const { return free_.empty() ? 0 : free_.rbegin()->first; }
  size_t used() const { return used_; }
  size_t peak() const { return peak_; }
  void reset_peak() { peak_ = used_; }
  size_t capacity() const { return cap_; }
  char* base() const { return base_; }
  bool owns(const void* p) const {
    const char* c = static_cast<const char*>(p);
    return base_ != nullptr && c >= base_ && c < base_ + cap_;
  }
  template <class F>
  void for_each_free(F&& f) const {
    for (auto& kv : free_) f(kv.second);
  }
  template <class F>
  void for_each_live(F&& f) const {
    for (auto& kv : live_) f(kv.second);
  }

 private:
  void clear() {
    Block* b = head_;
    while (b) {
      Block* n = b->next;
      delete b;
      b = n;
    }
    head_ = nullptr;
    free_.clear();
    live_.clear();
    used_ = peak_ = 0;
  }

  struct BySize {
    bool operator()(const std::pair<size_t, Block*>& a, const std::pair<size_t, Block*>& b) const {
      if (a.first != b.first) return a.first < b.first;
      // nullptr sorts first so lower_bound({size, nullptr}) is the first block of that size
      if (a.second == nullptr || b.second == nullptr) return a.second == nullptr && b.second != nullptr;
      return a.second->off < b.second->off;
    }
  };

  char* base_ = nullptr;
  size_t align_ = kAlign;

  void* fresh_ = nullptr;
  size_t cap_ = 0;
  Block* head_ = nullptr;
  std::set<std::pair<size_t, Block*>, BySize> free_;
  std::map<size_t, Block*> live_;
  size_t used_ = 0, peak_ = 0;
};

}  // namespace lms
