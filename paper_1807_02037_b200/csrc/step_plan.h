// Static placement of one training step's device allocations.
//
// A swapped training step allocates the same sizes in the same order every
// iteration.  After one recorded step the pool knows each allocation's size
// and lifetime (alloc event .. free event on one logical clock), so it can
// place all of them once, offline, inside one contiguous region: no
// fragmentation, no page moves, no allocator search on the hot path.  The
// reference's memory model is the same idea in discrete form: residency is
// a per-tensor interval between "alloc at op start" and "free at refcount 0"
// (sim.py:116-124, :193-211).
//
// Placement is greedy: items in a priority order, each at the lowest offset
// (or in the tightest gap) whose range is free for its whole lifetime.  Three
// orders (size descending; size x lifetime descending; allocation order) x
// two gap rules are tried and the smallest region wins.  No
// CUDA here, so it is unit-testable on the host (lms_plan_solve).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace lms {

struct PlanItem {
  uint64_t size = 0;   // bytes (already rounded to the pool's granule)
  int64_t t0 = 0;      // alloc event
  int64_t t1 = -1;     // free event; < 0: outlives the step (not planned)
  int64_t t1_logical = -1;  // the owner's free; t1 may be later (a swap-out still read it)
  uint64_t off = 0;    // placement (valid when planned)
  bool planned = false;
};

namespace detail {

// best_fit=false: lowest offset whose gap fits; true: the smallest gap that
// fits (ties: lowest offset), the region top counting as an unbounded gap
inline uint64_t place_in_order(std::vector<PlanItem>& it, const std::vector<size_t>& order,
                               std::vector<uint64_t>* offs, bool best_fit = false) {
  offs->assign(it.size(), 0);
  std::vector<size_t> placed;
  placed.reserve(order.size());
  std::vector<std::pair<uint64_t, uint64_t>> busy;
  uint64_t top = 0;
  for (size_t i : order) {
    busy.clear();
    for (size_t j : placed)
      if (it[j].t0 < it[i].t1 && it[i].t0 < it[j].t1) busy.emplace_back((*offs)[j], (*offs)[j] + it[j].size);
    std::sort(busy.begin(), busy.end());
    uint64_t off = 0;
    if (!best_fit) {
      for (auto& b : busy) {
        if (b.first >= off + it[i].size) break;  // the gap before b fits
        off = std::max(off, b.second);
      }
    } else {
      uint64_t cur = 0, best_gap = UINT64_MAX;
      bool found = false;
      for (auto& b : busy) {
        if (b.first > cur) {
          const uint64_t gap = b.first - cur;
          if (gap >= it[i].size && gap < best_gap) {
            best_gap = gap;
            off = cur;
            found = true;
          }
        }
        cur = std::max(cur, b.second);
      }
      if (!found) off = cur;  // above everything live at the same time
    }
    (*offs)[i] = off;
    top = std::max(top, off + it[i].size);
    placed.push_back(i);
  }
  return top;
}

}  // namespace detail

inline uint64_t plan_live_peak(const std::vector<PlanItem>& it);

// Place every item with t1 >= 0; returns the region size.  Items with t1 < 0
// stay unplanned (the dynamic pool serves them).  After the deterministic
// orders, randomized restarts (size keys jittered by x0.6..1.4, fixed seed)
// run until the region fits `target` or reaches the live-bytes lower bound,
// at most `restarts` times: first-fit by size gets stuck when a short-lived
// giant (a cuDNN workspace) takes the bottom of a tall stack.
inline uint64_t plan_place(std::vector<PlanItem>& it, uint64_t target = 0, int restarts = 400) {
  std::vector<size_t> idx;
  for (size_t i = 0; i < it.size(); ++i) {
    it[i].planned = it[i].t1 >= 0 && it[i].t1 > it[i].t0;
    if (it[i].planned) idx.push_back(i);
  }
  if (idx.empty()) return 0;
  auto by_size = idx;
  std::stable_sort(by_size.begin(), by_size.end(), [&](size_t a, size_t b) {
    if (it[a].size != it[b].size) return it[a].size > it[b].size;
    return it[a].t0 < it[b].t0;
  });
  auto by_area = idx;
  std::stable_sort(by_area.begin(), by_area.end(), [&](size_t a, size_t b) {
    const double aa = double(it[a].size) * double(it[a].t1 - it[a].t0);
    const double bb = double(it[b].size) * double(it[b].t1 - it[b].t0);
    if (aa != bb) return aa > bb;
    return it[a].t0 < it[b].t0;
  });
  auto by_time = idx;  // allocation order (what a dynamic allocator sees)
  std::vector<std::vector<size_t>*> orders = {&by_size, &by_area, &by_time};
  uint64_t best_size = UINT64_MAX;
  std::vector<uint64_t> best, o;
  for (auto* ord : orders)
    for (bool bf : {false, true}) {
      const uint64_t sz = detail::place_in_order(it, *ord, &o, bf);
      if (sz < best_size) {
        best_size = sz;
        best.swap(o);
      }
    }
  const uint64_t bound = plan_live_peak(it);
  uint64_t rng = 0x9E3779B97F4A7C15ull;
  auto next = [&rng] {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
  };
  std::vector<double> key(it.size());
  auto by_jit = idx;
  for (int r = 0; r < restarts && best_size > bound && best_size > target; ++r) {
    for (size_t i : idx) key[i] = double(it[i].size) * (0.6 + 0.8 * double(next() >> 11) * 0x1.0p-53);
    std::stable_sort(by_jit.begin(), by_jit.end(), [&](size_t a, size_t b) { return key[a] > key[b]; });
    const uint64_t sz = detail::place_in_order(it, by_jit, &o, false);
    if (sz < best_size) {
      best_size = sz;
      best.swap(o);
    }
  }
  for (size_t i : idx) it[i].off = best[i];
  return best_size;
}

// Lifetimes end at the physical release (after the block's swap-out copy).
// When that placement does not fit in `room`, pull each end toward the
// owner's free (t1 = t1_logical + a (t1 - t1_logical)) and bisect on a: a
// block reused before its copy finished makes the next allocation wait for
// that copy on replay, which is the price of fitting.  Returns the region
// size and the blend used via *alpha.
inline uint64_t plan_place_fit(std::vector<PlanItem>& it, uint64_t room, double* alpha) {
  std::vector<int64_t> phys(it.size());
  for (size_t i = 0; i < it.size(); ++i) phys[i] = it[i].t1;
  auto blend = [&](double a) {
    for (size_t i = 0; i < it.size(); ++i) {
      const int64_t lg = it[i].t1_logical;
      it[i].t1 = (phys[i] >= 0 && lg >= 0 && lg < phys[i])
                     ? lg + int64_t(a * double(phys[i] - lg) + 0.5) : phys[i];
      if (it[i].t1 >= 0 && it[i].t1 <= it[i].t0) it[i].t1 = it[i].t0 + 1;
    }
  };
  *alpha = 1.0;
  uint64_t r = plan_place(it, room);
  if (r <= room) return r;
  double lo = 0.0, hi = 1.0;
  blend(0.0);
  r = plan_place(it, room);
  if (r > room) {
    *alpha = 0.0;
    return r;  // does not fit even with the owners' frees
  }
  std::vector<PlanItem> best = it;
  uint64_t best_r = r;
  for (int k = 0; k < 6; ++k) {
    const double mid = 0.5 * (lo + hi);
    blend(mid);
    r = plan_place(it, room);
    if (r <= room) {
      lo = mid;
      best = it;
      best_r = r;
    } else {
      hi = mid;
    }
  }
  it = best;
  *alpha = lo;
  return best_r;
}

// max over time of the bytes live at once: the lower bound any placement
// of these lifetimes needs
inline uint64_t plan_live_peak(const std::vector<PlanItem>& it) {
  std::vector<std::pair<int64_t, int64_t>> ev;
  for (auto& x : it)
    if (x.planned) {
      ev.emplace_back(x.t0, int64_t(x.size));
      ev.emplace_back(x.t1, -int64_t(x.size));
    }
  std::sort(ev.begin(), ev.end());  // frees (negative) sort first at equal times
  int64_t cur = 0, peak = 0;
  for (auto& e : ev) {
    cur += e.second;
    peak = std::max(peak, cur);
  }
  return uint64_t(peak);
}

}  // namespace lms
