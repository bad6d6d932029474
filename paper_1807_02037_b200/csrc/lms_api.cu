// liblms.so: device pool, pinned host pool and swap engine behind the C ABI
// declared in include/lms.h.  See that header for the reference semantics
// each entry point implements.
//
// Streams: each context owns one D2H and one H2D stream (the simulator's
// per-direction channels, sim.py:284-322); with overlap_transfers=0 both
// directions share one stream (the shared "xfer" channel, sim.py:287-290).
// The compute stream belongs to the caller (PyTorch's current stream).
//
// Device blocks are tagged with the stream that last used them.  A block is
// handed to another stream only after that stream waits on an event
// recorded on the previous owner, and a block read by an in-flight swap-out
// is not reused before the copy completes (sim.py:205-211).

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <sys/syscall.h>
#include <unistd.h>

#include "../../include/lms.h"
#include "arena.h"
#include "kernels.cuh"
#include "vmm_pool.h"
#include "step_plan.h"

namespace lms {

static thread_local std::string g_err;
static lms_ctx* g_global = nullptr;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(LMS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

static void* const kFresh = reinterpret_cast<void*>(~uintptr_t(0));

// NVTX ranges on the host side of every swap/pool call (no-ops unless a tool
// such as nsys is attached): the timeline shows when each transfer was issued
// and where allocations waited for swap-out copies
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ---------------------------------------------------------------------------
// NUMA: pinned host chunks are placed on the GPU's own NUMA node (its PCIe
// root complex), so each DP rank's swap traffic stays on its socket's memory
// controllers.  Raw syscalls: libnuma is not a dependency.

int device_numa_node(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  for (char* q = bus; *q; ++q) *q = char(tolower(*q));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

// prefer `node` for the pages this thread faults in while in scope
struct NumaPrefer {
  bool on = false;
  explicit NumaPrefer(int node) {
    if (node < 0 || node >= 64) return;
    unsigned long mask = 1ul << node;
    on = syscall(SYS_set_mempolicy, 1 /* MPOL_PREFERRED */, &mask, 64) == 0;
  }
  ~NumaPrefer() {
    if (on) syscall(SYS_set_mempolicy, 0 /* MPOL_DEFAULT */, nullptr, 0);
  }
};

// NUMA node holding the page at p (-1 if unknown)
int page_node(const void* p) {
  int node = -1;
  if (syscall(SYS_get_mempolicy, &node, nullptr, 0, const_cast<void*>(p), 3 /* MPOL_F_NODE|MPOL_F_ADDR */) != 0)
    return -1;
  return node;
}

struct OomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// events: disable-timing events recycled through a free list

class EventPool {
 public:
  cudaEvent_t get(bool timing = false) {
    auto& fl = timing ? timed_ : plain_;
    if (!fl.empty()) {
      cudaEvent_t e = fl.back();
      fl.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
    return e;
  }
  void put(cudaEvent_t e, bool timing = false) {
    if (e) (timing ? timed_ : plain_).push_back(e);
  }
  ~EventPool() {
    for (auto e : plain_) cudaEventDestroy(e);
    for (auto e : timed_) cudaEventDestroy(e);
  }

 private:
  std::vector<cudaEvent_t> plain_, timed_;
};

// shared, reference-counted event (one swap-out event may hold a block and
// gate several swap-ins)
struct SharedEv {
  cudaEvent_t e = nullptr;
  int refs = 0;
};

struct XferRec {
  int64_t handle_id;
  int direction, codec;
  uint64_t logical, wire;
  cudaEvent_t start, end;
};

// a device allocation on its way back to the pool
struct DevBlk {
  char* base = nullptr;
  size_t size = 0;
  Block* blk = nullptr;
  void* stream = nullptr;   // freeing stream
  uint64_t seq = 0;         // that stream's clock at the free
};

}  // namespace lms

using namespace lms;

struct lms_handle {
  int64_t id = 0;
  int ndim = 0;
  int64_t sizes[LMS_MAX_DIMS] = {};
  int64_t strides[LMS_MAX_DIMS] = {};
  int elem = 0;
  int64_t numel = 0;
  int64_t span = 0;        // storage elements covered by the view
  bool packed = false;     // host copy is contiguous (view was not dense)
  int codec = LMS_CODEC_RAW_CE;
  char* host = nullptr;
  size_t host_bytes = 0;   // reserved
  uint64_t logical = 0;    // tensor bytes
  uint64_t wire = 0;       // bytes that crossed PCIe on swap-out (bound until known)
  SharedEv* out_done = nullptr;
  cudaEvent_t in_ready = nullptr;  // last swap-in (H2D is in order: covers all reads)
  bool wire_known = true;          // false until a ZVC header has been read back
  int64_t rec_out = -1;            // index of the swap-out timing record
  int64_t rec_in = -1;             // index of the last swap-in timing record
  uint64_t rec_gen = 0;            // trace generation the record indices belong to
  std::vector<int64_t> zvc_in_recs;  // ZVC swap-in records issued before the size was known
  uint64_t zvc_in_pending = 0;       // such swap-ins not yet in the h2d wire counter
  bool released = false;
};

struct lms_ctx {
  lms_config_t cfg{};
  std::mutex mu;
  int device = 0;
  int num_sms = 148;
  cudaStream_t d2h = nullptr, h2d = nullptr;
  void* home = nullptr;  // compute stream (immediate reuse)
  EventPool events;

  // device pool: VA arenas over CUDA virtual memory, physical pages under the budget
  VmmPool* vmm = nullptr;
  size_t limit = 0;
  size_t alloc_bytes = 0, alloc_peak = 0;   // live block bytes (the model's residency)
  uint64_t n_reclaims = 0, n_device_syncs = 0;
  size_t mapped_peak = 0;
  std::unordered_map<char*, std::vector<SharedEv*>> holds;  // block base -> pending readers
  std::unordered_map<char*, std::vector<void*>> rec_streams;  // block base -> extra streams using it
  std::vector<DevBlk> deferred;                             // freed, waiting for their holds
  size_t deferred_bytes = 0;

  // static step plan (step_plan.h): record one step's allocations, place them
  // once inside a single region, replay the placement on later steps
  struct PlanFreed {
    size_t off, size;
    void* stream;
    uint64_t seq;
    char* base;   // key of the block's swap-out holds
    size_t item;  // plan item it served
    bool released;  // its swap-out copies were seen finished
  };
  struct StepPlan {
    int mode = LMS_PLAN_OFF;
    bool ready = false;
    std::vector<PlanItem> items;
    std::unordered_map<char*, size_t> rec_live;   // record: ptr -> item
    std::unordered_map<char*, size_t> rec_held;   // record: freed, waiting for its swap-out copy
    int64_t clock = 0;
    Block* region = nullptr;
    char* base = nullptr;
    size_t size = 0, lower_bound = 0, solved = 0;
    double alpha = 1.0;   // lifetime blend the placement needed (1 = physical releases)
    std::vector<int64_t> t1_phys;  // recorded physical release events (before any blend)
    std::vector<PlanItem> refine;  // REFINE: lifetimes observed while replaying
    int64_t rclock = 0;
    uint64_t refinements = 0;
    size_t cursor = 0;
    size_t resyncs = 0;   // this replay's allocations off the recorded sequence
    bool diverged = false;
    std::map<size_t, std::pair<size_t, size_t>> live;  // off -> (size, item)
    std::vector<PlanFreed> freed;
    size_t live_bytes = 0;
    uint64_t hits = 0, dynamic = 0, diverged_steps = 0;
  } plan;

  // pinned host pool: chunks, each an arena
  struct Chunk {
    char* base;
    Arena* arena;
  };
  std::vector<Chunk> chunks;
  size_t host_reserved = 0;
  size_t host_used = 0, host_peak = 0;
  int numa_node = -1;                // the GPU's NUMA node (pinned chunks prefer it)
  uint64_t chunks_on_node = 0;       // pinned chunks whose pages landed there
  std::vector<lms_handle*> zombie;   // released handles waiting for H2D reads
  std::vector<lms_handle*> zvc_open; // ZVC swap-outs whose compressed size is not yet known

  // stats
  lms_stats_t st{};
  int64_t next_id = 1;

  // timing
  cudaEvent_t epoch = nullptr;
  std::vector<XferRec> recs;
  uint64_t trace_gen = 0;   // bumped by lms_trace_clear
  int use_bulk = 1;         // ZVC kernels move chunks with cp.async.bulk (LMS_ZVC_BULK=0: STG/LDG)
  int zc_ctas = 0;          // CTAs of the zero-copy (host-side) kernels
  int zc_dec_ctas = 0;      // ... of the zero-copy decode (LMS_ZC_DEC_CTAS)
  int use_tma_pack = 1;     // pack/unpack of rows layouts through tensor maps (LMS_TMA_PACK=0: SIMT)
  // strided (non-dense) swaps: packed/unpacked in HBM by the TMA kernels through a
  // staging block owned by each copy channel, moved by the copy engine
  // (LMS_STAGE_STRIDED=0: SIMT kernels straight to/from pinned memory)
  int stage_strided = 1;
  int enc_per_sm = 1;       // resident encode CTAs per SM (occupancy API)
  char* stage[2] = {nullptr, nullptr};   // [0] D2H channel, [1] H2D channel
  // consumer reached its wait (event on the consumer stream) vs swap-in record
  std::vector<std::pair<cudaEvent_t, int64_t>> waits;
};

namespace {

// -------------------------------------------------------------------------
// device pool internals (caller holds ctx->mu)

void retire_event(lms_ctx* c, SharedEv* ev) {
  if (--ev->refs == 0) {
    c->events.put(ev->e);
    delete ev;
  }
}

// drop completed holds; true if the block has none left
bool holds_clear(lms_ctx* c, char* base) {
  auto it = c->holds.find(base);
  if (it == c->holds.end()) return true;
  auto& v = it->second;
  size_t w = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    if (cudaEventQuery(v[i]->e) == cudaSuccess) retire_event(c, v[i]);
    else v[w++] = v[i];
  }
  v.resize(w);
  if (w == 0) {
    c->holds.erase(it);
    return true;
  }
  return false;
}

// give a freed block back to the pool
void release_block(lms_ctx* c, const DevBlk& d) {
  if (c->plan.mode == LMS_PLAN_RECORD) {
    // a recorded block's lifetime ends when its memory is really reusable:
    // after its swap-out copy, not at the logical free
    auto& P = c->plan;
    auto it = P.rec_held.find(d.base);
    if (it != P.rec_held.end()) {
      P.items[it->second].t1 = P.clock++;
      P.rec_held.erase(it);
    }
  }
  c->alloc_bytes -= d.size;
  c->vmm->free(d.blk, d.stream, d.seq);
}

void reap_deferred(lms_ctx* c, bool block) {
  size_t w = 0;
  for (size_t i = 0; i < c->deferred.size(); ++i) {
    DevBlk& d = c->deferred[i];
    if (block) {
      auto it = c->holds.find(d.base);
      if (it != c->holds.end())
        for (auto* ev : it->second) cudaEventSynchronize(ev->e);
    }
    if (holds_clear(c, d.base)) {
      c->deferred_bytes -= d.size;
      release_block(c, d);
    } else {
      c->deferred[w++] = d;
    }
  }
  c->deferred.resize(w);
}

// wait for deferred frees oldest first, one block at a time, until `enough`
// holds.  Waiting for every pending swap-out at once would drain the D2H
// channel and leave the link idle while the compute stream produces the next
// tensor; waiting for just the oldest keeps the later copies queued.
template <class F>
void reap_until(lms_ctx* c, F enough) {
  reap_deferred(c, false);
  if (c->deferred.empty() || enough()) return;
  NvtxRange nv("lms:alloc_wait_swap_out");
  const auto t0 = std::chrono::steady_clock::now();
  while (!c->deferred.empty() && !enough()) {
    auto it = c->holds.find(c->deferred.front().base);
    if (it != c->holds.end())
      for (auto* ev : it->second) cudaEventSynchronize(ev->e);
    c->n_device_syncs++;
    reap_deferred(c, false);
  }
  c->st.alloc_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void stream_wait_on(lms_ctx* c, void* waiter, void* owner) {
  cudaEvent_t e = c->events.get();
  cudaEventRecord(e, static_cast<cudaStream_t>(owner));
  cudaStreamWaitEvent(static_cast<cudaStream_t>(waiter), e, 0);
  c->events.put(e);  // the wait captured the record; the event may be re-recorded later
  c->st.n_cross_stream_waits++;
}

int ensure_pool(lms_ctx* c) {
  if (c->vmm) return LMS_OK;
  size_t limit = c->cfg.device_reserve ? c->cfg.device_reserve : c->cfg.device_limit;
  if (limit == 0) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    limit = fr > (size_t(2) << 30) ? fr - (size_t(2) << 30) : fr / 2;
  }
  auto* v = new VmmPool();
  std::string err;
  size_t page = size_t(64) << 20;
  if (const char* pm = getenv("LMS_PAGE_MB")) page = size_t(std::max(2, atoi(pm))) << 20;
  if (!v->init(c->device, limit, kFresh, &err, page)) {
    delete v;
    return fail(LMS_E_CUDA, "device pool: " + err);
  }
  c->vmm = v;
  c->limit = c->cfg.device_limit && c->cfg.device_limit < v->limit_bytes() ? c->cfg.device_limit
                                                                            : v->limit_bytes();
  return LMS_OK;
}

int oom(lms_ctx* c, size_t size, const std::string& why) {
  VmmPool& v = *c->vmm;
  c->st.n_oom++;
  if (getenv("LMS_DEBUG_OOM")) {
    std::vector<uint64_t> sz;
    v.for_each_live([&](uint64_t s) { sz.push_back(s); });
    std::sort(sz.begin(), sz.end(), std::greater<uint64_t>());
    fprintf(stderr, "[lms] OOM wanting %zu B: %zu live blocks, deferred %zu B, largest:", size, sz.size(),
            c->deferred_bytes);
    for (size_t i = 0; i < sz.size() && i < 16; ++i) fprintf(stderr, " %.0fM", sz[i] / 1048576.0);
    fprintf(stderr, "\n");
  }
  char buf[320];
  snprintf(buf, sizeof buf,
           "LMS_OOM: device budget exhausted allocating %zu bytes (live %zu, mapped %zu, limit %zu, "
           "page %zu): %s", size, c->alloc_bytes, v.mapped_bytes(), c->limit, v.page(), why.c_str());
  return fail(LMS_E_OOM, buf);
}

// ---- static step plan -------------------------------------------------------

bool in_plan(lms_ctx* c, const void* p) {
  const char* q = static_cast<const char*>(p);
  return c->plan.base && q >= c->plan.base && q < c->plan.base + c->plan.size;
}

size_t dev_in_use(lms_ctx* c) {
  return c->alloc_bytes - (c->plan.region ? c->plan.size : 0) + c->plan.live_bytes;
}

void note_peak(lms_ctx* c) { c->alloc_peak = std::max(c->alloc_peak, dev_in_use(c)); }

// wait until no hold on `base` is pending (its swap-out copies finished)
void drain_holds(lms_ctx* c, char* base) {
  while (!holds_clear(c, base)) {
    auto it = c->holds.find(base);
    if (it == c->holds.end()) break;
    for (auto* ev : it->second) cudaEventSynchronize(ev->e);
    c->n_device_syncs++;
  }
}

constexpr size_t kPlanMaxResyncs = 32;
constexpr size_t kPlanSkipAhead = 8;   // recorded allocations a replay may skip in a row

// replay: serve the next recorded allocation from its planned offset.
// Returns 1 when this request is not planned (the dynamic pool serves it).
int plan_alloc(lms_ctx* c, size_t rsize, void* stream, void** out) {
  auto& P = c->plan;
  if (P.cursor >= P.items.size()) {
    P.diverged = true;
    return 1;
  }
  size_t idx = P.cursor++;
  if (P.items[idx].size != rsize) {
    // an allocation the recording did not make (a DDP buffer broadcast's
    // staging tensor, say) is served by the dynamic pool and the cursor stays;
    // recorded allocations this step did not make (up to kPlanSkipAhead in a
    // row) are stepped over when a following item matches.  Past
    // kPlanMaxResyncs per step the sequences differ.
    static const bool dbg = getenv("LMS_PLAN_DEBUG") != nullptr;
    if (dbg)
      fprintf(stderr, "[lms plan] item %zu: recorded %llu B, requested %zu B (resync %zu)\n", idx,
              (unsigned long long)P.items[idx].size, rsize, P.resyncs);
    if (P.resyncs >= kPlanMaxResyncs) {
      P.diverged = true;  // the step allocates differently from the recorded one
      P.diverged_steps++;
      return 1;
    }
    P.resyncs++;
    size_t j = idx + 1;
    const size_t end = std::min(P.items.size(), idx + 1 + kPlanSkipAhead);
    while (j < end && P.items[j].size != rsize) ++j;
    if (j < end) {
      idx = j;              // items idx..j-1 were not requested this step
      P.cursor = j + 1;
    } else {
      P.cursor = idx;       // an extra allocation: retry item idx on the next request
      return 1;
    }
  }
  const PlanItem& it = P.items[idx];
  if (!it.planned) return 1;
  const size_t lo = it.off, hi = it.off + it.size;
  // a planned block still live over this range means the sequences drifted
  auto nx = P.live.lower_bound(lo);
  if (nx != P.live.end() && nx->first < hi) {
    P.diverged = true;
    P.diverged_steps++;
    return 1;
  }
  if (nx != P.live.begin()) {
    auto pv = std::prev(nx);
    if (pv->first + pv->second.first > lo) {
      P.diverged = true;
      P.diverged_steps++;
      return 1;
    }
  }
  // earlier users of the range: swap-out copies still reading it, and work
  // on another stream, must finish first (the dynamic pool's rules)
  const auto t0 = std::chrono::steady_clock::now();
  bool waited = false;
  size_t w = 0;
  const bool refine = P.mode == LMS_PLAN_REFINE;
  for (size_t i = 0; i < P.freed.size(); ++i) {
    lms_ctx::PlanFreed& f = P.freed[i];
    if (refine && !f.released && holds_clear(c, f.base)) {
      f.released = true;  // seen released before this allocation
      P.refine[f.item].t1 = P.rclock;
    }
    const bool overlap = f.off < hi && lo < f.off + f.size;
    if (overlap) {
      if (!holds_clear(c, f.base)) {
        drain_holds(c, f.base);
        waited = true;
      }
      if (f.stream != stream && !c->vmm->clocks_.passed(f.stream, f.seq)) {
        c->vmm->clocks_.device_wait(stream, f.stream, f.seq);
        c->st.n_cross_stream_waits++;
      }
    }
    if (refine && !f.released && holds_clear(c, f.base)) {
      f.released = true;  // this allocation waited for it
      P.refine[f.item].t1 = P.rclock;
    }
    // keep entries whose range may still be busy for some later request (and,
    // when refining, whose release has not been seen yet)
    if (!(holds_clear(c, f.base) && c->vmm->clocks_.passed(f.stream, f.seq)) || (refine && !f.released))
      P.freed[w++] = f;
  }
  P.freed.resize(w);
  if (refine) P.refine[idx].t0 = P.rclock++;
  if (waited)
    c->st.alloc_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  P.live[lo] = {it.size, idx};
  P.live_bytes += it.size;
  P.hits++;
  c->st.n_alloc++;
  note_peak(c);
  *out = P.base + lo;
  return LMS_OK;
}

// a freed block recorded on other streams is held until the work enqueued
// there by now completes (the CUDA caching allocator's recordStream rule)
void apply_recorded_streams(lms_ctx* c, char* base) {
  auto it = c->rec_streams.find(base);
  if (it == c->rec_streams.end()) return;
  for (void* s : it->second) {
    auto* ev = new SharedEv();
    ev->e = c->events.get();
    ev->refs = 1;
    cudaEventRecord(ev->e, static_cast<cudaStream_t>(s));
    c->holds[base].push_back(ev);
  }
  c->rec_streams.erase(it);
}

void plan_free(lms_ctx* c, void* ptr, void* stream) {
  auto& P = c->plan;
  const size_t off = static_cast<char*>(ptr) - P.base;
  auto it = P.live.find(off);
  if (it == P.live.end()) return;
  const size_t size = it->second.first;
  const size_t item = it->second.second;
  apply_recorded_streams(c, static_cast<char*>(ptr));
  P.live.erase(it);
  P.live_bytes -= size;
  bool released = true;
  if (P.mode == LMS_PLAN_REFINE) {
    P.refine[item].t1_logical = P.rclock++;
    released = holds_clear(c, static_cast<char*>(ptr));
    if (released) P.refine[item].t1 = P.refine[item].t1_logical;
  }
  P.freed.push_back({off, size, stream, c->vmm->clocks_.stamp(stream), static_cast<char*>(ptr), item, released});
  c->st.n_free++;
}

// returns LMS_OK and *out, or LMS_E_OOM.  The budget is on live pages; when
// it is short only because freed blocks still wait for their swap-out copies
// the call blocks until those copies land (this is what throttles a forward
// pass that outruns the D2H channel).
int dev_alloc_locked(lms_ctx* c, size_t size, void* stream, void** out) {
  int rc = ensure_pool(c);
  if (rc) return rc;
  VmmPool& v = *c->vmm;
  reap_deferred(c, false);
  const size_t rsize = Arena::round(size);
  const bool replaying = c->plan.mode == LMS_PLAN_REPLAY || c->plan.mode == LMS_PLAN_REFINE;
  if (replaying && c->plan.ready && !c->plan.diverged) {
    rc = plan_alloc(c, rsize, stream, out);
    if (rc == LMS_OK) return LMS_OK;
  }
  if (replaying) c->plan.dynamic++;
  // the budget is on live bytes; the non-deferred live set only shrinks by
  // frees the caller has not made yet, so fail at once if it plus the request
  // is over (cuDNN's plan loop probes oversized workspaces and expects a
  // quick OOM); if deferred frees are in the way, wait for their copies
  if (c->alloc_bytes - c->deferred_bytes + rsize > c->limit)
    return oom(c, size, "live set plus request exceeds the budget");
  if (c->alloc_bytes + rsize > c->limit) reap_until(c, [&] { return c->alloc_bytes + rsize <= c->limit; });
  if (c->alloc_bytes + rsize > c->limit) return oom(c, size, "live set plus request exceeds the budget");
  // a mapped range first; if freed blocks still wait for their swap-out
  // copies, wait for those (oldest first: the D2H channel stays busy) before
  // paying for page moves (driver calls on the host thread)
  std::string err;
  Block* b = v.alloc(size, stream, false, &err, false);
  while (!b && !c->deferred.empty()) {
    const size_t before = c->deferred.size();
    reap_until(c, [&] { return c->deferred.size() < before; });
    err.clear();
    b = v.alloc(size, stream, false, &err, false);
  }
  if (!b) {
    err.clear();
    b = v.alloc(size, stream, false, &err, true);
  }
  if (!b) {
    err.clear();
    b = v.alloc(size, stream, true, &err, true);
  }
  if (!b) return oom(c, size, err);
  // a range last used by another stream: wait for that use on the device
  if (b->tag != kFresh && b->tag != stream && !v.idle(b)) {
    v.clocks_.device_wait(stream, b->tag, b->seq);
    c->st.n_cross_stream_waits++;
  }
  b->tag = stream;
  c->st.n_alloc++;
  c->alloc_bytes += b->size;
  note_peak(c);
  c->mapped_peak = std::max(c->mapped_peak, v.mapped_bytes());
  *out = v.ptr(b);
  if (c->plan.mode == LMS_PLAN_RECORD) {
    auto& P = c->plan;
    PlanItem it;
    it.size = rsize;
    it.t0 = P.clock++;
    P.rec_live[static_cast<char*>(*out)] = P.items.size();
    P.items.push_back(it);
  }
  return LMS_OK;
}

bool find_dev(lms_ctx* c, const void* ptr, bool exact, DevBlk* d) {
  if (in_plan(c, ptr)) {
    auto& P = c->plan;
    const size_t off = static_cast<const char*>(ptr) - P.base;
    auto it = P.live.upper_bound(off);
    if (it == P.live.begin()) return false;
    --it;
    if (off >= it->first + it->second.first || (exact && off != it->first)) return false;
    d->base = P.base + it->first;
    d->size = it->second.first;
    d->blk = nullptr;
    return true;
  }
  Block* b = exact ? c->vmm->find(ptr) : c->vmm->containing(ptr);
  if (!b) return false;
  d->base = c->vmm->ptr(b);
  d->size = b->size;
  d->blk = b;
  return true;
}

int dev_free_locked(lms_ctx* c, void* ptr, void* stream) {
  if (!ptr) return LMS_OK;
  if (!c->vmm || !c->vmm->owns(ptr)) return fail(LMS_E_INVALID, "lms_dev_free: pointer not from the device pool");
  if (in_plan(c, ptr)) {
    plan_free(c, ptr, stream);
    return LMS_OK;
  }
  if (c->plan.mode == LMS_PLAN_RECORD) {
    auto& P = c->plan;
    auto it = P.rec_live.find(static_cast<char*>(ptr));
    if (it != P.rec_live.end()) {
      P.items[it->second].t1_logical = P.clock++;
      P.rec_held[static_cast<char*>(ptr)] = it->second;  // t1 set in release_block
      P.rec_live.erase(it);
    }
  }
  DevBlk d;
  if (!find_dev(c, ptr, true, &d)) return fail(LMS_E_INVALID, "lms_dev_free: not a live allocation");
  apply_recorded_streams(c, d.base);
  d.stream = stream;
  d.seq = c->vmm->clocks_.stamp(stream);
  c->st.n_free++;
  if (!holds_clear(c, d.base)) {
    c->deferred.push_back(d);
    c->deferred_bytes += d.size;
    c->st.n_deferred_frees++;
    return LMS_OK;
  }
  release_block(c, d);
  return LMS_OK;
}

// -------------------------------------------------------------------------
// host pool internals (caller holds ctx->mu)

int host_alloc_locked(lms_ctx* c, size_t size, void** out) {
  size_t need = Arena::round(size);
  for (auto& ch : c->chunks) {
    Block* b = ch.arena->alloc(need);
    if (b) {
      *out = ch.base + b->off;
      c->host_used += b->size;
      c->host_peak = std::max(c->host_peak, c->host_used);
      return LMS_OK;
    }
  }
  size_t grow = std::max(need, c->cfg.host_chunk ? c->cfg.host_chunk : (size_t(1) << 30));
  if (c->cfg.host_limit) {
    if (c->host_reserved + need > c->cfg.host_limit)
      return fail(LMS_E_HOST_OOM, "pinned host limit reached (" + std::to_string(c->host_reserved) + " of " +
                                      std::to_string(c->cfg.host_limit) + " bytes pinned)");
    grow = std::min(grow, c->cfg.host_limit - c->host_reserved);
  }
  void* p = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e;
  {
    NumaPrefer np(c->numa_node);
    e = cudaHostAlloc(&p, grow, cudaHostAllocPortable | cudaHostAllocMapped);
  }
  if (e == cudaSuccess && c->numa_node >= 0 && page_node(p) == c->numa_node) c->chunks_on_node++;
  c->st.host_grow_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->st.n_host_grow++;
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(LMS_E_HOST_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  }
  auto* a = new Arena();
  a->init(static_cast<char*>(p), grow);
  c->chunks.push_back({static_cast<char*>(p), a});
  c->host_reserved += grow;
  Block* b = a->alloc(need);
  *out = static_cast<char*>(p) + b->off;
  c->host_used += b->size;
  c->host_peak = std::max(c->host_peak, c->host_used);
  return LMS_OK;
}

int host_free_locked(lms_ctx* c, void* ptr) {
  for (auto& ch : c->chunks) {
    if (ch.arena->owns(ptr)) {
      Block* b = ch.arena->find_live(static_cast<char*>(ptr) - ch.base);
      if (!b) return fail(LMS_E_INVALID, "lms_host_free: not a live allocation");
      c->host_used -= b->size;
      ch.arena->release(b);
      return LMS_OK;
    }
  }
  return fail(LMS_E_INVALID, "lms_host_free: pointer not from the host pool");
}

// bytes a finished encoded stream occupies on the wire: header + tile table +
// each tile's chunk (host-readable stream; `bound` if it is not one)
uint64_t zvc_wire_bytes(const char* enc, uint64_t bound) {
  const ZvcHeader* hd = reinterpret_cast<const ZvcHeader*>(enc);
  if (hd->magic != kZvcMagic) return bound;
  const ZvcTile* tab = reinterpret_cast<const ZvcTile*>(enc + hd->table_pos);
  uint64_t b = 64 + hd->ntiles * 8;
  for (uint64_t t = 0; t < hd->ntiles; ++t) b += tab[t].bytes;
  return b;
}

bool is_zvc(int codec) { return codec == LMS_CODEC_ZVC || codec == LMS_CODEC_ZX; }

// learn the compressed size of finished ZVC swap-outs (table in pinned memory)
void account_zvc(lms_ctx* c) {
  size_t w = 0;
  for (size_t i = 0; i < c->zvc_open.size(); ++i) {
    lms_handle* h = c->zvc_open[i];
    if (cudaEventQuery(h->out_done->e) != cudaSuccess) {
      c->zvc_open[w++] = h;
      continue;
    }
    h->wire = zvc_wire_bytes(h->host, h->host_bytes);
    h->wire_known = true;
    c->st.d2h_wire_bytes += h->wire;
    c->st.h2d_wire_bytes += h->wire * h->zvc_in_pending;
    h->zvc_in_pending = 0;
    if (h->rec_gen == c->trace_gen) {
      if (h->rec_out >= 0 && size_t(h->rec_out) < c->recs.size()) c->recs[h->rec_out].wire = h->wire;
      for (int64_t r : h->zvc_in_recs)
        if (r >= 0 && size_t(r) < c->recs.size()) c->recs[r].wire = h->wire;
    }
    h->zvc_in_recs.clear();
  }
  c->zvc_open.resize(w);
}

void reap_zombies(lms_ctx* c) {
  account_zvc(c);
  size_t w = 0;
  for (size_t i = 0; i < c->zombie.size(); ++i) {
    lms_handle* h = c->zombie[i];
    bool busy = h->in_ready && cudaEventQuery(h->in_ready) != cudaSuccess;
    if (h->out_done && cudaEventQuery(h->out_done->e) != cudaSuccess) busy = true;
    if (busy || !h->wire_known) {
      c->zombie[w++] = h;
      continue;
    }
    if (h->out_done) retire_event(c, h->out_done);
    if (h->in_ready) c->events.put(h->in_ready);
    if (h->host) host_free_locked(c, h->host);
    delete h;
  }
  c->zombie.resize(w);
}

// -------------------------------------------------------------------------
// launch helpers

int sm_grid(lms_ctx* c, int64_t work_items, int per_cta) {
  int64_t want = (work_items + per_cta - 1) / per_cta;
  int cap = c->cfg.sm_ctas > 0 ? c->cfg.sm_ctas : c->num_sms * 4;
  if (want < 1) want = 1;
  return int(std::min<int64_t>(want, cap));
}

bool dense_layout(int ndim, const int64_t* sizes, const int64_t* strides, int64_t* span_out,
                  int64_t* numel_out) {
  int64_t numel = 1, span = 1;
  for (int k = 0; k < ndim; ++k) {
    numel *= sizes[k];
    if (sizes[k] > 1) span += (sizes[k] - 1) * strides[k];
  }
  if (numel == 0) span = 0;
  *span_out = span;
  *numel_out = numel;
  return span <= numel;
}

void to_desc(Strided* d, int ndim, const int64_t* sizes, const int64_t* strides) {
  std::memset(d, 0, sizeof(*d));
  d->ndim = ndim;
  for (int k = 0; k < ndim; ++k) {
    d->sizes[k] = sizes[k];
    d->strides[k] = strides[k];
  }
}

// ---- TMA pack/unpack --------------------------------------------------------

bool is_host_ptr(const void* p);

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

constexpr int kTmaStages = 4;
constexpr uint32_t kTmaBoxTarget = 16384;

// Rows layouts (the strided side's innermost dim has unit stride) through
// tensor maps.  sizes/strides: row-major, squeezed; strides are the strided
// side's (elements).  Returns 1 when the layout does not qualify (the caller
// uses the SIMT kernels), 0 on launch, <0 on error.
template <bool PACK>
int launch_tma_rows(lms_ctx* c, char* dst, const char* src, int nd, const int64_t* sizes, const int64_t* strides,
                    int elem, cudaStream_t s) {
  if (!c->use_tma_pack || nd < 1 || strides[nd - 1] != 1) return 1;
  if (reinterpret_cast<uintptr_t>(dst) % 16 || reinterpret_cast<uintptr_t>(src) % 16) return 1;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return 1;
  // merge row-major dims the strided side keeps adjacent
  int64_t ms[LMS_MAX_DIMS + 1], mz[LMS_MAX_DIMS + 1];
  int n = 0;
  for (int k = 0; k < nd; ++k) {
    if (n > 0 && ms[n - 1] == strides[k] * sizes[k]) {
      mz[n - 1] *= sizes[k];
      ms[n - 1] = strides[k];
    } else {
      mz[n] = sizes[k];
      ms[n] = strides[k];
      ++n;
    }
  }
  if (n > 5) return 1;
  cuuint64_t gdim[5], sstr[4], cstr[4];
  cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) gdim[i] = i < n ? cuuint64_t(mz[n - 1 - i]) : 1;
  uint64_t cacc = uint64_t(elem);
  for (int i = 1; i < 5; ++i) {
    cacc *= gdim[i - 1];
    cstr[i - 1] = cacc;
    sstr[i - 1] = i < n ? uint64_t(ms[n - 1 - i]) * elem : (i == 1 ? cacc : sstr[i - 2] * gdim[i - 1]);
  }
  for (int i = 0; i < 4; ++i) {
    if (gdim[i] > (uint64_t(1) << 32) || cstr[i] % 16 || sstr[i] % 16 || cstr[i] >= (uint64_t(1) << 40) ||
        sstr[i] >= (uint64_t(1) << 40))
      return 1;
  }
  // box: innermost up to 256 elements (a 16 B multiple), then fill ~16 KiB
  uint32_t b0 = uint32_t(std::min<uint64_t>(gdim[0], 256));
  const uint32_t q = 16 / std::min(elem, 16);
  b0 = (b0 + q - 1) / q * q;
  if (b0 > 256) return 1;
  box[0] = b0;
  uint64_t bytes = uint64_t(b0) * elem;
  for (int i = 1; i < 5; ++i) {
    uint64_t room = std::max<uint64_t>(1, kTmaBoxTarget / bytes);
    box[i] = uint32_t(std::min<uint64_t>({gdim[i], room, 256}));
    bytes *= box[i];
  }
  CUtensorMapDataType dt = elem == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                           : elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                       : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  CUtensorMap ms_map, mc_map;  // strided side, contiguous side
  const char* strided = PACK ? src : dst;
  const char* contig = PACK ? dst : src;
  if (enc(&ms_map, dt, 5, const_cast<char*>(strided), gdim, sstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS ||
      enc(&mc_map, dt, 5, const_cast<char*>(contig), gdim, cstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
    return 1;
  TmaBoxGrid g{};
  g.total = 1;
  for (int i = 0; i < 5; ++i) {
    g.box[i] = box[i];
    g.nbox[i] = uint32_t((gdim[i] + box[i] - 1) / box[i]);
    g.total *= g.nbox[i];
  }
  const int grid = int(std::min<uint64_t>(g.total, uint64_t(c->num_sms) * 4));
  const uint32_t box_bytes = uint32_t(bytes);
  const uint32_t stage_bytes = (box_bytes + 1023) / 1024 * 1024;
  tma_copy_kernel<kTmaStages><<<grid, 32, size_t(kTmaStages) * stage_bytes, s>>>(
      PACK ? ms_map : mc_map, PACK ? mc_map : ms_map, g, box_bytes, stage_bytes);
  c->st.kernel_launches++;
  CK(cudaGetLastError());
  return 0;
}

// warps per CTA of the TMA transpose (each holds 4 tiles of (128/E) x 128 B)
template <int E>
constexpr int tt_warps() { return E == 1 ? 2 : 4; }
constexpr int kTmaTWarps = 4;

template <int E>
size_t tma_transpose_smem() { return 1024 + size_t(tt_warps<E>()) * 4 * (128 / E) * 128; }

// Transposed layouts (the strided side's unit-stride dim `cd` is not its last
// dim) through 128 B-swizzled tensor maps.  Same contract as launch_tma_rows.
template <bool PACK>
int launch_tma_transpose(lms_ctx* c, char* dst, const char* src, int nd, const int64_t* sizes,
                         const int64_t* strides, int elem, cudaStream_t s) {
  if (!c->use_tma_pack || nd < 2) return 1;
  if (reinterpret_cast<uintptr_t>(dst) % 16 || reinterpret_cast<uintptr_t>(src) % 16) return 1;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return 1;
  const int last = nd - 1;
  int cd = -1;
  for (int k = 0; k < last; ++k)
    if (strides[k] == 1) cd = k;
  if (cd < 0 || strides[last] == 1) return 1;
  // contiguous-side (row-major) strides
  int64_t cst[LMS_MAX_DIMS + 1];
  {
    int64_t acc = 1;
    for (int k = nd - 1; k >= 0; --k) {
      cst[k] = acc;
      acc *= sizes[k];
    }
  }
  // batch dims (all but cd and last), innermost first, merged where both sides allow
  int64_t bz[LMS_MAX_DIMS], bs_s[LMS_MAX_DIMS], bs_c[LMS_MAX_DIMS];
  int nb = 0;
  for (int k = last - 1; k >= 0; --k) {
    if (k == cd) continue;
    if (nb > 0 && bs_s[nb - 1] * bz[nb - 1] == strides[k] && bs_c[nb - 1] * bz[nb - 1] == cst[k]) {
      bz[nb - 1] *= sizes[k];
      continue;
    }
    bz[nb] = sizes[k];
    bs_s[nb] = strides[k];
    bs_c[nb] = cst[k];
    ++nb;
  }
  if (nb > 3) return 1;
  const uint32_t T = 128 / elem;
  // strided map: d0 = cd (unit), d1 = last; contiguous map: d0 = last (unit), d1 = cd
  cuuint64_t gs[5], gc[5], ss[4], sc[4];
  gs[0] = sizes[cd];
  gs[1] = sizes[last];
  ss[0] = uint64_t(strides[last]) * elem;
  gc[0] = sizes[last];
  gc[1] = sizes[cd];
  sc[0] = uint64_t(cst[cd]) * elem;
  for (int i = 0; i < 3; ++i) {
    const bool real = i < nb;
    gs[2 + i] = gc[2 + i] = real ? cuuint64_t(bz[i]) : 1;
    ss[1 + i] = real ? uint64_t(bs_s[i]) * elem : ss[i] * gs[1 + i];
    sc[1 + i] = real ? uint64_t(bs_c[i]) * elem : sc[i] * gc[1 + i];
  }
  for (int i = 0; i < 4; ++i)
    if (ss[i] % 16 || sc[i] % 16 || ss[i] >= (uint64_t(1) << 40) || sc[i] >= (uint64_t(1) << 40)) return 1;
  for (int i = 0; i < 5; ++i)
    if (gs[i] > (uint64_t(1) << 32)) return 1;
  CUtensorMapDataType dt = elem == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                           : elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                       : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  cuuint32_t box[5] = {T, T, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  const char* strided = PACK ? src : dst;
  const char* contig = PACK ? dst : src;
  CUtensorMap m_s, m_c;
  if (enc(&m_s, dt, 5, const_cast<char*>(strided), gs, ss, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS ||
      enc(&m_c, dt, 5, const_cast<char*>(contig), gc, sc, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
    return 1;
  // the box grid walks the LOAD map's dims
  const cuuint64_t* gl = PACK ? gs : gc;
  TmaBoxGrid g{};
  g.total = 1;
  for (int i = 0; i < 5; ++i) {
    g.box[i] = box[i];
    g.nbox[i] = uint32_t((gl[i] + box[i] - 1) / box[i]);
    g.total *= g.nbox[i];
  }
  const CUtensorMap& ld = PACK ? m_s : m_c;
  const CUtensorMap& st = PACK ? m_c : m_s;
  static const int per_sm = getenv("LMS_TMA_T_CTAS") ? std::max(1, atoi(getenv("LMS_TMA_T_CTAS"))) : 12;
  const int grid = int(std::min<uint64_t>((g.total + kTmaTWarps - 1) / kTmaTWarps, uint64_t(c->num_sms) * per_sm));
  switch (elem) {
    case 1: tma_transpose_kernel<1, tt_warps<1>()><<<grid, 32 * tt_warps<1>(), tma_transpose_smem<1>(), s>>>(ld, st, g); break;
    case 2: tma_transpose_kernel<2, tt_warps<2>()><<<grid, 32 * tt_warps<2>(), tma_transpose_smem<2>(), s>>>(ld, st, g); break;
    case 4: tma_transpose_kernel<4, tt_warps<4>()><<<grid, 32 * tt_warps<4>(), tma_transpose_smem<4>(), s>>>(ld, st, g); break;
    default: tma_transpose_kernel<8, tt_warps<8>()><<<grid, 32 * tt_warps<8>(), tma_transpose_smem<8>(), s>>>(ld, st, g); break;
  }
  c->st.kernel_launches++;
  CK(cudaGetLastError());
  return 0;
}

// pack (dst contiguous) or unpack (dst strided); either side may be mapped host
// memory.  `mem`: 0 both sides in HBM, 1 one side is host memory, -1 unknown
// (the public entry points: one cudaPointerGetAttributes per side)
enum { kMemDevice = 0, kMemHost = 1, kMemUnknown = -1 };
template <bool PACK>
int launch_layout(lms_ctx* c, char* dst, const char* src, int ndim, const int64_t* sizes_in,
                  const int64_t* strides_in, int elem, cudaStream_t s, int mem) {
  int64_t sizes[LMS_MAX_DIMS + 1], strides[LMS_MAX_DIMS + 1];
  // squeeze size-1 dims; widen 16-byte elements into two 8-byte words
  int nd = 0;
  for (int k = 0; k < ndim; ++k) {
    if (sizes_in[k] == 1) continue;
    sizes[nd] = sizes_in[k];
    strides[nd] = strides_in[k];
    ++nd;
  }
  if (elem == 16) {
    for (int k = 0; k < nd; ++k) strides[k] *= 2;
    sizes[nd] = 2;
    strides[nd] = 1;
    ++nd;
    elem = 8;
  }
  if (nd == 0) {
    sizes[0] = 1;
    strides[0] = 1;
    nd = 1;
  }
  if (nd > LMS_MAX_DIMS) return fail(LMS_E_INVALID, "too many dimensions");
  if (elem != 1 && elem != 2 && elem != 4 && elem != 8) return fail(LMS_E_INVALID, "unsupported element size");
  int64_t numel = 1;
  for (int k = 0; k < nd; ++k) numel *= sizes[k];
  if (numel == 0) return LMS_OK;
  Strided d;
  to_desc(&d, nd, sizes, strides);
#define DISPATCH_E(KERNEL, ...)                                                       \
  switch (elem) {                                                                     \
    case 1: KERNEL<PACK, 1><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                  \
    case 2: KERNEL<PACK, 2><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                  \
    case 4: KERNEL<PACK, 4><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                  \
    default: KERNEL<PACK, 8><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                 \
  }
  const int last = nd - 1;
  if (mem == kMemUnknown) mem = (is_host_ptr(dst) || is_host_ptr(src)) ? kMemHost : kMemDevice;
  if (mem == kMemDevice) {
    int rc = strides[last] == 1 ? launch_tma_rows<PACK>(c, dst, src, nd, sizes, strides, elem, s)
                                : launch_tma_transpose<PACK>(c, dst, src, nd, sizes, strides, elem, s);
    if (rc <= 0) return rc;
  }
  if (strides[last] == 1) {
    int64_t row = sizes[last], rows = numel / row;
    bool vec = (row * elem) % 16 == 0 && (reinterpret_cast<uintptr_t>(dst) % 16 == 0) &&
               (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    for (int k = 0; k < last && vec; ++k) vec = (strides[k] * elem) % 16 == 0;
    int grid = sm_grid(c, rows, 8);
    if (vec) {
      switch (elem) {
        case 1: rows_kernel<PACK, true, 1><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        case 2: rows_kernel<PACK, true, 2><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        case 4: rows_kernel<PACK, true, 4><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        default: rows_kernel<PACK, true, 8><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
      }
    } else {
      switch (elem) {
        case 1: rows_kernel<PACK, false, 1><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        case 2: rows_kernel<PACK, false, 2><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        case 4: rows_kernel<PACK, false, 4><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
        default: rows_kernel<PACK, false, 8><<<grid, 256, 0, s>>>(dst, src, d, rows, row); break;
      }
    }
  } else {
    int cd = -1;
    for (int k = 0; k < last; ++k)
      if (strides[k] == 1) cd = k;
    // the transpose kernel keeps in-tile offsets in 32 bits
    const bool small_strides = cd >= 0 && 31 * (strides[cd] + strides[last]) < (int64_t(1) << 31) &&
                               numel / sizes[cd] * 32 < (int64_t(1) << 31);
    if (cd >= 0 && sizes[cd] >= 8 && sizes[last] >= 8 && small_strides) {
      int64_t batches = numel / (sizes[cd] * sizes[last]);
      int64_t tiles = batches * ((sizes[cd] + 31) / 32) * ((sizes[last] + 31) / 32);
      int grid = sm_grid(c, tiles, 1);
      DISPATCH_E(transpose_kernel, dst, src, d, cd, batches);
    } else {
      int grid = sm_grid(c, numel, 256 * 4);
      DISPATCH_E(generic_kernel, dst, src, d, numel);
    }
  }
#undef DISPATCH_E
  c->st.kernel_launches++;
  CK(cudaGetLastError());
  return LMS_OK;
}

constexpr size_t kStageBytes = size_t(32) << 20;

// the channel's staging block (allocated once from the pool, owned by that
// stream: stream order alone keeps chunk k+1's pack behind chunk k's copy)
char* stage_block(lms_ctx* c, int dir) {
  cudaStream_t s = dir == 0 ? c->d2h : c->h2d;
  if (dir == 1 && c->h2d == c->d2h) dir = 0;   // one shared channel: one block
  if (!c->stage[dir]) {
    if (!c->vmm) return nullptr;   // a context without a device pool does not grow one for this
    void* p = nullptr;
    const std::string keep = g_err;
    // a one-off allocation: not part of any recorded or replayed step plan
    const int mode = c->plan.mode;
    c->plan.mode = LMS_PLAN_OFF;
    const int rc = dev_alloc_locked(c, kStageBytes, s, &p);
    c->plan.mode = mode;
    if (rc != LMS_OK) {
      g_err = keep;
      return nullptr;   // no room: the SIMT zero-copy path serves this swap
    }
    c->stage[dir] = static_cast<char*>(p);
  }
  return c->stage[dir];
}

// dims before the first one longer than 1 are trivial: slabs along it are
// contiguous ranges of the packed layout
bool slab_dim(int ndim, const int64_t* sizes, int elem, int* k0, uint64_t* row_bytes) {
  int k = 0;
  while (k < ndim - 1 && sizes[k] == 1) ++k;
  uint64_t rb = uint64_t(elem);
  for (int j = k + 1; j < ndim; ++j) rb *= uint64_t(sizes[j]);
  *k0 = k;
  *row_bytes = rb;
  return ndim > 0 && rb <= kStageBytes;
}

// strided swap-out: TMA pack of slabs into the D2H staging block + copy-engine
// D2H of each.  Returns 1 (nothing enqueued) when staging cannot serve it.
int staged_pack_d2h(lms_ctx* c, char* host, const char* src, int ndim, const int64_t* sizes,
                    const int64_t* strides, int elem, cudaStream_t s) {
  int k0;
  uint64_t row;
  if (!c->stage_strided || !slab_dim(ndim, sizes, elem, &k0, &row)) return 1;
  char* stg = stage_block(c, 0);
  if (!stg) return 1;
  const int64_t per = int64_t(kStageBytes / row);
  int64_t sz[LMS_MAX_DIMS];
  std::memcpy(sz, sizes, sizeof(int64_t) * ndim);
  for (int64_t a = 0; a < sizes[k0]; a += per) {
    sz[k0] = std::min(per, sizes[k0] - a);
    int rc = launch_layout<true>(c, stg, src + a * strides[k0] * elem, ndim, sz, strides, elem, s, kMemDevice);
    if (rc) return rc;
    CK(cudaMemcpyAsync(host + a * row, stg, uint64_t(sz[k0]) * row, cudaMemcpyDeviceToHost, s));
  }
  return 0;
}

// strided swap-in into `dst` (layout dst_strides): copy-engine H2D of slabs of
// the packed host copy into the H2D staging block + TMA unpack of each
int staged_unpack_h2d(lms_ctx* c, char* dst, const char* host, int ndim, const int64_t* sizes,
                      const int64_t* dst_strides, int elem, cudaStream_t s) {
  int k0;
  uint64_t row;
  if (!c->stage_strided || !slab_dim(ndim, sizes, elem, &k0, &row)) return 1;
  char* stg = stage_block(c, 1);
  if (!stg) return 1;
  const int64_t per = int64_t(kStageBytes / row);
  int64_t sz[LMS_MAX_DIMS];
  std::memcpy(sz, sizes, sizeof(int64_t) * ndim);
  for (int64_t a = 0; a < sizes[k0]; a += per) {
    sz[k0] = std::min(per, sizes[k0] - a);
    CK(cudaMemcpyAsync(stg, host + a * row, uint64_t(sz[k0]) * row, cudaMemcpyHostToDevice, s));
    int rc = launch_layout<false>(c, dst + a * dst_strides[k0] * elem, stg, ndim, sz, dst_strides, elem, s,
                                  kMemDevice);
    if (rc) return rc;
  }
  return 0;
}

int launch_copy(lms_ctx* c, char* dst, const char* src, size_t bytes, cudaStream_t s) {
  size_t n16 = bytes / 16;
  if (n16) {
    int grid = sm_grid(c, int64_t(n16), 512 * 4);
    copy16_kernel<<<grid, 512, 0, s>>>(reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src),
                                       int64_t(n16));
    c->st.kernel_launches++;
  }
  if (bytes % 16) {
    copy_tail_kernel<<<1, 32, 0, s>>>(dst + n16 * 16, src + n16 * 16, int64_t(bytes % 16));
    c->st.kernel_launches++;
  }
  CK(cudaGetLastError());
  return LMS_OK;
}

bool is_host_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;  // unknown to CUDA: treat as host (the SIMT kernels handle both)
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

int launch_zvc_encode(lms_ctx* c, const uint32_t* src, uint64_t nwords, char* out, cudaStream_t s,
                      bool to_host, bool allow_exp) {
  const uint64_t ntiles = zvc_tiles(nwords);
  // one pass: HBM-side encodes take the whole GPU; encodes into pinned memory
  // take enough CTAs to keep the link busy without crowding the compute stream
  // HBM side: exactly the CTAs that are resident at once (a grid-stride loop
  // with a partial second wave would leave most SMs idle at the end)
  int grid = int(std::min<int64_t>(int64_t(ntiles), int64_t(c->num_sms) * c->enc_per_sm));
  if (to_host) grid = int(std::min<int64_t>(int64_t(ntiles), c->zc_ctas));
  if (allow_exp)
    zvc_encode_kernel<true><<<std::max(grid, 1), 256, kZvcEncSmemBytes, s>>>(src, nwords, out, c->use_bulk);
  else
    zvc_encode_kernel<false><<<std::max(grid, 1), 256, kZvcEncSmemBytes, s>>>(src, nwords, out, c->use_bulk);
  c->st.kernel_launches++;
  CK(cudaGetLastError());
  return LMS_OK;
}

int launch_zvc_decode(lms_ctx* c, const char* enc, uint64_t nwords, uint32_t* dst, cudaStream_t s,
                      bool from_host) {
  int grid = sm_grid(c, int64_t(zvc_tiles(nwords)), 1);
  if (from_host)
    grid = int(std::min<int64_t>(int64_t(zvc_tiles(nwords)), c->zc_dec_ctas > 0 ? c->zc_dec_ctas : c->zc_ctas));
  zvc_decode_kernel<<<std::max(grid, 1), 256, kZvcSmemBytes, s>>>(enc, nwords, dst, c->use_bulk);
  c->st.kernel_launches++;
  CK(cudaGetLastError());
  return LMS_OK;
}

// timing keeps the most recent transfers only: past kMaxRecs the oldest
// finished half is dropped (their events go back to the pool) and the record
// indices handles hold are invalidated through trace_gen
constexpr size_t kMaxRecs = size_t(1) << 17;

void trim_records(lms_ctx* c) {
  size_t k = 0;
  const size_t half = c->recs.size() / 2;
  while (k < half && cudaEventQuery(c->recs[k].end) == cudaSuccess) ++k;
  if (k == 0) return;
  for (size_t i = 0; i < k; ++i) {
    c->events.put(c->recs[i].start, true);
    c->events.put(c->recs[i].end, true);
  }
  c->recs.erase(c->recs.begin(), c->recs.begin() + k);
  size_t w = 0;
  for (size_t i = 0; i < c->waits.size(); ++i) {
    auto wt = c->waits[i];
    if (wt.second < int64_t(k)) {
      c->events.put(wt.first, true);
      continue;
    }
    wt.second -= int64_t(k);
    c->waits[w++] = wt;
  }
  c->waits.resize(w);
  c->trace_gen++;
}

void timing_begin(lms_ctx* c, cudaStream_t s, cudaEvent_t* start) {
  *start = nullptr;
  if (!c->cfg.timing) return;
  if (c->recs.size() >= kMaxRecs) trim_records(c);
  *start = c->events.get(true);
  cudaEventRecord(*start, s);
}

void timing_end(lms_ctx* c, cudaStream_t s, cudaEvent_t start, lms_handle* h, int dir, uint64_t logical,
                uint64_t wire) {
  if (!c->cfg.timing || !start) return;
  cudaEvent_t end = c->events.get(true);
  cudaEventRecord(end, s);
  c->recs.push_back({h->id, dir, h->codec, logical, wire, start, end});
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" {

const char* lms_last_error(void) { return g_err.c_str(); }
const char* lms_version(void) { return "lms 0.1.0 sm_100a"; }

int lms_default_config(lms_config_t* cfg) {
  if (!cfg) return fail(LMS_E_INVALID, "null config");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->host_chunk = size_t(1) << 30;
  cfg->overlap_transfers = 1;
  return LMS_OK;
}

int lms_create(const lms_config_t* cfg, lms_ctx** out) {
  if (!cfg || !out) return fail(LMS_E_INVALID, "null argument");
  auto* c = new lms_ctx();
  c->cfg = *cfg;
  c->device = cfg->device;
  c->limit = cfg->device_limit;
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(LMS_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  c->numa_node = device_numa_node(c->device);
  if (const char* v = getenv("LMS_NUMA")) {
    if (atoi(v) < 0) c->numa_node = -1;   // LMS_NUMA=-1: no placement policy
  }
  // zero-copy kernels: one CTA per SM by default (each keeps a 16 KiB chunk
  // in flight on the link), overridable for tuning
  c->zc_ctas = cfg->sm_ctas > 0 ? cfg->sm_ctas : c->num_sms;
  if (const char* v = getenv("LMS_ZC_CTAS")) c->zc_ctas = std::max(1, atoi(v));
  // decode CTAs (LMS_ZC_DEC_CTAS): 37 / 56 / 74 / 100 / 148 all keep the H2D
  // wire rate; at 908 the step measured 334.5 / 335.3 / 354.5 / 338.2 / 337.3
  // img/s, within the run-to-run spread of the swapped bytes (52.0 - 54.5 GB
  // per direction), so the decode keeps the encode's count
  c->zc_dec_ctas = c->zc_ctas;
  if (const char* v = getenv("LMS_ZC_DEC_CTAS")) c->zc_dec_ctas = std::max(1, atoi(v));
  if (const char* v = getenv("LMS_ZVC_BULK")) c->use_bulk = atoi(v) != 0;
  if (const char* v = getenv("LMS_TMA_PACK")) c->use_tma_pack = atoi(v) != 0;
  if (const char* v = getenv("LMS_STAGE_STRIDED")) c->stage_strided = atoi(v) != 0;
  cudaFuncSetAttribute(tma_copy_kernel<kTmaStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kTmaStages * int(kTmaBoxTarget) * 2);
  cudaFuncSetAttribute(tma_transpose_kernel<1, tt_warps<1>()>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(tma_transpose_smem<1>()));
  cudaFuncSetAttribute(tma_transpose_kernel<2, tt_warps<2>()>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(tma_transpose_smem<2>()));
  cudaFuncSetAttribute(tma_transpose_kernel<4, tt_warps<4>()>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(tma_transpose_smem<4>()));
  cudaFuncSetAttribute(tma_transpose_kernel<8, tt_warps<8>()>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(tma_transpose_smem<8>()));
  cudaFuncSetAttribute(zvc_encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kZvcEncSmemBytes);
  cudaFuncSetAttribute(zvc_encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kZvcEncSmemBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->enc_per_sm, zvc_encode_kernel<true>, 256, kZvcEncSmemBytes);
  c->enc_per_sm = std::max(1, c->enc_per_sm);
  cudaFuncSetAttribute(zvc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kZvcSmemBytes);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // transfers get the higher priority so their small kernels are not starved
  if (cudaStreamCreateWithPriority(&c->d2h, cudaStreamNonBlocking, hi) != cudaSuccess) {
    delete c;
    return fail(LMS_E_CUDA, "stream creation failed");
  }
  if (cfg->overlap_transfers) {
    cudaStreamCreateWithPriority(&c->h2d, cudaStreamNonBlocking, hi);
  } else {
    c->h2d = c->d2h;
  }
  if (cfg->device_reserve || cfg->device_limit) {
    int rc = ensure_pool(c);
    if (rc) {
      delete c;
      return rc;
    }
  }
  if (cfg->host_reserve) {
    void* p = nullptr;
    size_t keep = c->cfg.host_chunk;
    c->cfg.host_chunk = cfg->host_reserve;
    int rc = host_alloc_locked(c, 1, &p);
    c->cfg.host_chunk = keep;
    if (rc) {
      delete c;
      return rc;
    }
    host_free_locked(c, p);
  }
  c->epoch = c->events.get(true);
  cudaEventRecord(c->epoch, c->d2h);
  *out = c;
  return LMS_OK;
}

int lms_destroy(lms_ctx* c) {
  if (!c) return LMS_OK;
  cudaDeviceSynchronize();
  {
    std::lock_guard<std::mutex> g(c->mu);
    reap_zombies(c);
  }
  if (g_global == c) g_global = nullptr;
  for (auto& ch : c->chunks) {
    cudaFreeHost(ch.base);
    delete ch.arena;
  }
  delete c->vmm;
  if (c->h2d && c->h2d != c->d2h) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  delete c;
  return LMS_OK;
}

int lms_set_global(lms_ctx* c) {
  g_global = c;
  return LMS_OK;
}
lms_ctx* lms_get_global(void) { return g_global; }

int lms_set_home_stream(lms_ctx* c, void* s) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  c->home = s;
  return LMS_OK;
}

int lms_set_limit(lms_ctx* c, size_t limit) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  if (limit == 0) limit = c->cfg.device_reserve ? c->cfg.device_reserve : c->limit;
  c->cfg.device_limit = limit;
  if (c->vmm) {
    // physical pages are fixed at creation; the budget on live pages moves
    c->limit = std::min(limit, c->vmm->limit_bytes());
  } else {
    c->limit = limit;
  }
  return LMS_OK;
}

int lms_reset_peaks(lms_ctx* c) {
  std::lock_guard<std::mutex> g(c->mu);
  c->alloc_peak = c->alloc_bytes;
  c->mapped_peak = c->vmm ? c->vmm->mapped_bytes() : 0;
  c->host_peak = c->host_used;
  return LMS_OK;
}

int lms_set_tuning(lms_ctx* c, int zc_ctas, int use_bulk, int use_tma_pack) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  if (zc_ctas > 0) c->zc_ctas = c->zc_dec_ctas = zc_ctas;
  if (use_bulk >= 0) c->use_bulk = use_bulk != 0;
  if (use_tma_pack >= 0) c->use_tma_pack = use_tma_pack != 0;
  return LMS_OK;
}

int lms_get_streams(lms_ctx* c, void** d2h, void** h2d) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  if (d2h) *d2h = c->d2h;
  if (h2d) *h2d = c->h2d;
  return LMS_OK;
}

int lms_dev_alloc(lms_ctx* c, size_t size, void* stream, void** out) {
  if (!c || !out) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  return dev_alloc_locked(c, size, stream, out);
}

int lms_dev_free(lms_ctx* c, void* ptr, void* stream) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  return dev_free_locked(c, ptr, stream);
}

int lms_dev_hold_until(lms_ctx* c, const void* ptr, void* stream) {
  if (!c || !ptr) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->vmm || !c->vmm->owns(ptr)) return LMS_OK;  // not ours: nothing to hold
  DevBlk d;
  if (!find_dev(c, ptr, false, &d)) return fail(LMS_E_INVALID, "lms_dev_hold_until: pointer not in a live block");
  auto* ev = new SharedEv();
  ev->e = c->events.get();
  ev->refs = 1;
  CK(cudaEventRecord(ev->e, static_cast<cudaStream_t>(stream)));
  c->holds[d.base].push_back(ev);
  return LMS_OK;
}

int lms_plan_begin(lms_ctx* c, int mode) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  if (mode != LMS_PLAN_RECORD && mode != LMS_PLAN_REPLAY && mode != LMS_PLAN_REFINE && mode != LMS_PLAN_OFF)
    return fail(LMS_E_INVALID, "bad plan mode");
  std::lock_guard<std::mutex> g(c->mu);
  int rc = ensure_pool(c);
  if (rc) return rc;
  auto& P = c->plan;
  if (mode == LMS_PLAN_RECORD) {
    if (P.region) return fail(LMS_E_STATE, "a plan is active; lms_plan_reset first");
    P.items.clear();
    P.rec_live.clear();
    P.rec_held.clear();
    P.clock = 0;
    P.ready = false;
  } else if (mode == LMS_PLAN_REPLAY || mode == LMS_PLAN_REFINE) {
    if (!P.ready) return fail(LMS_E_STATE, "no recorded plan");
    P.cursor = 0;
    P.resyncs = 0;
    P.diverged = false;
    if (mode == LMS_PLAN_REFINE) {
      P.refine = P.items;
      for (auto& x : P.refine) x.t0 = 0, x.t1 = -1, x.t1_logical = -1;
      P.rclock = 0;
      for (auto& f : P.freed) f.released = true;  // the previous step's frees are not this step's
    }
  }
  P.mode = mode;
  return LMS_OK;
}

int lms_plan_end(lms_ctx* c) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  auto& P = c->plan;
  const int mode = P.mode;
  P.mode = LMS_PLAN_OFF;
  if (mode == LMS_PLAN_REFINE) {
    // re-place with the lifetimes this replay step showed; adopt the new
    // placement only if it fits the region already held
    if (P.diverged || P.resyncs || !P.live.empty()) return LMS_OK;
    std::vector<PlanItem> nx = P.refine;
    for (size_t i = 0; i < nx.size(); ++i) {
      if (!P.items[i].planned) {
        nx[i].t1 = -1;  // served dynamically: stays so
        continue;
      }
      if (nx[i].t1 < 0) nx[i].t1 = P.rclock + 1;  // copy not seen finished within the step
      if (nx[i].t1_logical < 0) nx[i].t1_logical = nx[i].t1;
    }
    double alpha = 1.0;
    const uint64_t region = plan_place_fit(nx, P.size, &alpha);
    if (region <= P.size) {
      for (size_t f = 0; f < P.freed.size(); ++f) drain_holds(c, P.freed[f].base);
      CK(cudaDeviceSynchronize());   // old placement's users finished
      P.freed.clear();
      P.items.swap(nx);
      P.solved = region;
      P.alpha = alpha;
      P.lower_bound = plan_live_peak(P.items);
      P.refinements++;
    }
    return LMS_OK;
  }
  if (mode != LMS_PLAN_RECORD) return LMS_OK;
  NvtxRange nv("lms:plan_place");
  P.rec_live.clear();  // still live at the end: t1 < 0, served dynamically
  P.rec_held.clear();
  // room for the region: the budget minus what stays live across steps
  reap_until(c, [] { return false; });
  // in whole physical pages: those no live block touches (the region needs its
  // own pages), less one page for the dynamic pool's unplanned allocations
  const size_t free_pages = c->vmm->limit_pages() - std::min(c->vmm->limit_pages(), c->vmm->live_pages());
  const uint64_t room = free_pages > 1 ? uint64_t(free_pages - 1) * c->vmm->page() : 0;
  double alpha = 1.0;
  P.t1_phys.resize(P.items.size());
  for (size_t i = 0; i < P.items.size(); ++i) P.t1_phys[i] = P.items[i].t1;
  const uint64_t region = plan_place_fit(P.items, room, &alpha);
  P.lower_bound = plan_live_peak(P.items);
  P.solved = region;
  P.alpha = alpha;
  if (region == 0) return LMS_OK;
  // the region is one live block of the dynamic pool; it counts against the budget
  reap_until(c, [&] { return c->alloc_bytes + region <= c->limit; });
  if (c->alloc_bytes + region > c->limit)
    return oom(c, region, "step plan region does not fit next to the live set");
  std::string err;
  Block* b = c->vmm->alloc(region, c->home ? c->home : nullptr, true, &err);
  if (!b) return oom(c, region, "step plan region: " + err);
  // the region's earlier users (any stream) must be done before planned reuse
  CK(cudaDeviceSynchronize());
  b->tag = kFresh;
  c->alloc_bytes += b->size;
  P.region = b;
  P.base = c->vmm->ptr(b);
  P.size = b->size;
  P.live.clear();
  P.freed.clear();
  P.live_bytes = 0;
  P.ready = true;
  return LMS_OK;
}

int lms_plan_reset(lms_ctx* c) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  auto& P = c->plan;
  if (!P.live.empty()) return fail(LMS_E_STATE, "planned blocks are still live");
  if (P.region) {
    for (auto& f : P.freed) drain_holds(c, f.base);
    CK(cudaDeviceSynchronize());
    c->alloc_bytes -= P.region->size;
    c->vmm->free(P.region, nullptr, 0);
    P.region = nullptr;
  }
  P.base = nullptr;
  P.size = 0;
  P.freed.clear();
  P.items.clear();
  P.ready = false;
  P.mode = LMS_PLAN_OFF;
  return LMS_OK;
}

int lms_plan_clock(lms_ctx* c, int64_t* out) {
  if (!c || !out) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  *out = c->plan.mode == LMS_PLAN_RECORD ? c->plan.clock : -1;
  return LMS_OK;
}

int lms_plan_info(lms_ctx* c, lms_plan_info_t* out) {
  if (!c || !out) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  auto& P = c->plan;
  lms_plan_info_t r{};
  r.ready = P.ready;
  r.region_bytes = P.size;
  r.lower_bound_bytes = P.lower_bound;
  r.solved_bytes = P.solved;
  r.alpha = P.alpha;
  r.refinements = P.refinements;
  {
    const size_t lp = c->vmm ? c->vmm->live_pages() : 0, tp = c->vmm ? c->vmm->limit_pages() : 0;
    r.room_bytes = (tp > lp ? uint64_t(tp - lp) * c->vmm->page() : 0) + (P.region ? P.size : 0);
  }
  r.n_items = P.items.size();
  for (auto& it : P.items) r.n_planned += it.planned;
  r.hits = P.hits;
  r.dynamic = P.dynamic;
  r.diverged_steps = P.diverged_steps;
  *out = r;
  return LMS_OK;
}

int lms_plan_items(lms_ctx* c, uint64_t* sizes, int64_t* t_alloc, int64_t* t_free, int64_t* t_free_logical,
                   size_t cap, size_t* n) {
  if (!c || !n) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  auto& it = c->plan.items;
  for (size_t i = 0; i < it.size() && i < cap; ++i) {
    if (sizes) sizes[i] = it[i].size;
    if (t_alloc) t_alloc[i] = it[i].t0;
    if (t_free) t_free[i] = i < c->plan.t1_phys.size() ? c->plan.t1_phys[i] : it[i].t1;
    if (t_free_logical) t_free_logical[i] = it[i].t1_logical;
  }
  *n = it.size();
  return LMS_OK;
}

int lms_plan_solve(const uint64_t* sizes, const int64_t* t_alloc, const int64_t* t_free, size_t n,
                   uint64_t* offsets, uint64_t* region) {
  if ((n && (!sizes || !t_alloc || !t_free || !offsets)) || !region) return fail(LMS_E_INVALID, "null argument");
  std::vector<PlanItem> it(n);
  for (size_t i = 0; i < n; ++i) {
    it[i].size = sizes[i];
    it[i].t0 = t_alloc[i];
    it[i].t1 = t_free[i];
  }
  *region = plan_place(it);
  for (size_t i = 0; i < n; ++i) offsets[i] = it[i].planned ? it[i].off : UINT64_MAX;
  return LMS_OK;
}

int lms_dev_record_stream(lms_ctx* c, const void* ptr, void* stream) {
  if (!c || !ptr) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->vmm || !c->vmm->owns(ptr)) return LMS_OK;
  DevBlk d;
  if (!find_dev(c, ptr, false, &d)) return fail(LMS_E_INVALID, "lms_dev_record_stream: pointer not in a live block");
  auto& v = c->rec_streams[d.base];
  if (std::find(v.begin(), v.end(), stream) == v.end()) v.push_back(stream);
  return LMS_OK;
}

int lms_host_alloc(lms_ctx* c, size_t size, void** out) {
  if (!c || !out) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  return host_alloc_locked(c, size, out);
}

int lms_host_reserve(lms_ctx* c, size_t total) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  if (c->cfg.host_limit) total = std::min(total, c->cfg.host_limit);
  const size_t chunk = c->cfg.host_chunk ? c->cfg.host_chunk : (size_t(1) << 30);
  while (c->host_reserved < total) {
    const size_t grow = std::min(chunk, total - c->host_reserved);
    void* q = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e;
    {
      NumaPrefer np(c->numa_node);
      e = cudaHostAlloc(&q, grow, cudaHostAllocPortable | cudaHostAllocMapped);
    }
    if (e == cudaSuccess && c->numa_node >= 0 && page_node(q) == c->numa_node) c->chunks_on_node++;
    c->st.host_grow_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(LMS_E_HOST_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    c->st.n_host_grow++;
    auto* a = new Arena();
    a->init(static_cast<char*>(q), grow);
    c->chunks.push_back({static_cast<char*>(q), a});
    c->host_reserved += grow;
  }
  return LMS_OK;
}

int lms_host_free(lms_ctx* c, void* ptr) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  return host_free_locked(c, ptr);
}

int lms_swap_out(lms_ctx* c, const void* src, const int64_t* sizes, const int64_t* strides, int ndim,
                 int elem_size, void* producer_stream, int codec, lms_handle** out) {
  if (!c || !out || (ndim > 0 && (!sizes || !strides))) return fail(LMS_E_INVALID, "null argument");
  if (ndim < 0 || ndim > LMS_MAX_DIMS) return fail(LMS_E_INVALID, "ndim out of range");
  if (elem_size <= 0) return fail(LMS_E_INVALID, "elem_size must be positive");
  for (int k = 0; k < ndim; ++k)
    if (sizes[k] < 0 || strides[k] < 0) return fail(LMS_E_INVALID, "negative size or stride");
  std::lock_guard<std::mutex> g(c->mu);
  NvtxRange nv("lms:swap_out");
  reap_zombies(c);
  auto* h = new lms_handle();
  h->id = c->next_id++;
  h->ndim = ndim;
  h->elem = elem_size;
  for (int k = 0; k < ndim; ++k) {
    h->sizes[k] = sizes[k];
    h->strides[k] = strides[k];
  }
  bool dense = dense_layout(ndim, sizes, strides, &h->span, &h->numel);
  h->packed = !dense;
  h->logical = uint64_t(h->numel) * elem_size;
  const uint64_t stored = h->packed ? h->logical : uint64_t(h->span) * elem_size;
  const bool aligned = reinterpret_cast<uintptr_t>(src) % 16 == 0;
  if (codec < LMS_CODEC_RAW_CE || codec > LMS_CODEC_ZX) {
    delete h;
    return fail(LMS_E_INVALID, "unknown codec");
  }
  if (is_zvc(codec) && (h->packed || stored % 4 != 0 || !aligned)) codec = LMS_CODEC_RAW_SM;
  if (codec == LMS_CODEC_RAW_SM && !h->packed && !aligned) codec = LMS_CODEC_RAW_CE;
  // a strided view is packed on its way out: TMA into the D2H staging block +
  // copy engine when staging is available (decided below), else one SIMT pack
  // kernel straight into pinned memory
  if (h->packed) codec = LMS_CODEC_RAW_SM;
  h->codec = codec;
  h->host_bytes = is_zvc(codec) ? zvc_bound(stored / 4) : (stored ? stored : 16);
  int rc = host_alloc_locked(c, h->host_bytes, reinterpret_cast<void**>(&h->host));
  if (rc) {
    delete h;
    return rc;
  }
  // the D2H channel starts after the producer's enqueued work
  cudaStream_t s = c->d2h;
  stream_wait_on(c, s, producer_stream);
  c->st.n_cross_stream_waits--;  // the producer dependency is the swap edge, not a pool wait
  cudaEvent_t t0;
  timing_begin(c, s, &t0);
  if (stored) {
    if (codec == LMS_CODEC_RAW_CE) {
      CK(cudaMemcpyAsync(h->host, src, stored, cudaMemcpyDeviceToHost, s));
      h->wire = stored;
    } else if (codec == LMS_CODEC_RAW_SM) {
      if (h->packed) {
        rc = staged_pack_d2h(c, h->host, static_cast<const char*>(src), ndim, sizes, strides, elem_size, s);
        if (rc == 0)
          h->codec = LMS_CODEC_RAW_CE;   // packed in HBM, moved by the copy engine
        else if (rc == 1)
          rc = launch_layout<true>(c, h->host, static_cast<const char*>(src), ndim, sizes, strides, elem_size, s,
                                   kMemHost);
      } else {
        rc = launch_copy(c, h->host, static_cast<const char*>(src), stored, s);
      }
      h->wire = stored;
    } else {
      rc = launch_zvc_encode(c, static_cast<const uint32_t*>(src), stored / 4, h->host, s, true,
                             codec == LMS_CODEC_ZX);
      h->wire = h->host_bytes;  // upper bound until the tile table is readable
    }
    if (rc) {
      host_free_locked(c, h->host);
      delete h;
      return rc;
    }
  }
  h->out_done = new SharedEv();
  h->out_done->e = c->events.get();
  h->out_done->refs = 1;
  CK(cudaEventRecord(h->out_done->e, s));
  if (c->cfg.timing && t0) {
    h->rec_out = int64_t(c->recs.size());
    h->rec_gen = c->trace_gen;
  }
  timing_end(c, s, t0, h, 0, h->logical, h->wire);
  if (is_zvc(codec) && stored) {
    h->wire_known = false;
    c->zvc_open.push_back(h);
  }
  // hold the source block until the copy is done
  if (stored && c->vmm && c->vmm->owns(src)) {
    DevBlk d;
    if (find_dev(c, src, false, &d)) {
      h->out_done->refs++;
      c->holds[d.base].push_back(h->out_done);
    }
  }
  c->st.n_swap_out++;
  c->st.n_handles_live++;
  c->st.d2h_logical_bytes += h->logical;
  if (!is_zvc(codec)) c->st.d2h_wire_bytes += h->wire;
  *out = h;
  return LMS_OK;
}

int lms_swap_in(lms_ctx* c, lms_handle* h, void* dst, const int64_t* dst_strides, void* trigger_stream) {
  if (!c || !h) return fail(LMS_E_INVALID, "null argument");
  if (!dst && h->numel > 0) return fail(LMS_E_INVALID, "null destination");
  std::lock_guard<std::mutex> g(c->mu);
  NvtxRange nv("lms:swap_in");
  if (h->released) return fail(LMS_E_STATE, "swap_in of a released handle");
  cudaStream_t s = c->h2d;
  // gate: the control op (everything enqueued on the trigger stream) and the swap-out
  stream_wait_on(c, s, trigger_stream);
  c->st.n_cross_stream_waits--;
  CK(cudaStreamWaitEvent(s, h->out_done->e, 0));
  // ZVC: the exact compressed size is known if the swap-out already finished;
  // otherwise the H2D moves the worst-case bound (correct, just more bytes)
  account_zvc(c);
  bool natural = dst_strides == nullptr;
  if (!natural && !h->packed) {
    natural = true;
    for (int k = 0; k < h->ndim; ++k)
      if (h->sizes[k] > 1 && dst_strides[k] != h->strides[k]) natural = false;
  }
  if (!natural && h->packed) {
    // contiguous strides requested on a packed handle are its natural layout
    natural = true;
    int64_t acc = 1;
    for (int k = h->ndim - 1; k >= 0; --k) {
      if (h->sizes[k] > 1 && dst_strides[k] != acc) natural = false;
      acc *= h->sizes[k];
    }
  }
  const uint64_t stored = h->packed ? h->logical : uint64_t(h->span) * h->elem;
  cudaEvent_t t0;
  timing_begin(c, s, &t0);
  uint64_t wire = 0;
  int rc = LMS_OK;
  if (stored) {
    if (!natural) {
      // arbitrary destination layout: scatter straight out of pinned memory
      if (is_zvc(h->codec)) return fail(LMS_E_INVALID, "ZVC handles restore to their own layout");
      if (!h->packed)
        return fail(LMS_E_INVALID, "a dense view restores only into its own strides (pass NULL)");
      rc = staged_unpack_h2d(c, static_cast<char*>(dst), h->host, h->ndim, h->sizes, dst_strides, h->elem, s);
      if (rc == 1)
        rc = launch_layout<false>(c, static_cast<char*>(dst), h->host, h->ndim, h->sizes, dst_strides, h->elem, s,
                                  kMemHost);
      wire = stored;
    } else if (is_zvc(h->codec)) {
      // zero-copy: the decode kernel reads the compressed stream straight out
      // of pinned memory, so only the compressed bytes cross the link and no
      // device staging buffer is taken from the budget (copying the tile slots
      // through the H2D staging block with the copy engine and decoding in HBM
      // measured slower: 52.3 vs 57.7 GB/s of tensor for dense ZX streams)
      rc = launch_zvc_decode(c, h->host, stored / 4, static_cast<uint32_t*>(dst), s, true);
      wire = h->wire_known ? h->wire : 0;
    } else if (h->codec == LMS_CODEC_RAW_SM && reinterpret_cast<uintptr_t>(dst) % 16 == 0) {
      rc = launch_copy(c, static_cast<char*>(dst), h->host, stored, s);
      wire = stored;
    } else {
      CK(cudaMemcpyAsync(dst, h->host, stored, cudaMemcpyHostToDevice, s));
      wire = stored;
    }
  }
  if (rc) return rc;
  if (!h->in_ready) h->in_ready = c->events.get();
  CK(cudaEventRecord(h->in_ready, s));
  if (c->cfg.timing && t0) {
    h->rec_in = int64_t(c->recs.size());
    if (is_zvc(h->codec) && !h->wire_known) {
      if (h->rec_gen != c->trace_gen) h->zvc_in_recs.clear();
      h->zvc_in_recs.push_back(h->rec_in);
    }
    h->rec_gen = c->trace_gen;
  }
  timing_end(c, s, t0, h, 1, h->logical, wire);
  c->st.n_swap_in++;
  c->st.h2d_logical_bytes += h->logical;
  if (is_zvc(h->codec) && !h->wire_known)
    h->zvc_in_pending++;  // counted when the swap-out's header is readable
  else
    c->st.h2d_wire_bytes += wire;
  return LMS_OK;
}

int lms_swap_wait(lms_ctx* c, lms_handle* h, void* consumer_stream) {
  if (!c || !h) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  if (!h->in_ready) return fail(LMS_E_STATE, "swap_wait before swap_in");
  if (c->cfg.timing && h->rec_in >= 0 && h->rec_gen == c->trace_gen) {
    cudaEvent_t reach = c->events.get(true);
    CK(cudaEventRecord(reach, static_cast<cudaStream_t>(consumer_stream)));
    c->waits.push_back({reach, h->rec_in});
  }
  CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(consumer_stream), h->in_ready, 0));
  return LMS_OK;
}

int lms_swap_out_done(lms_ctx* c, lms_handle* h) {
  if (!c || !h) return fail(LMS_E_INVALID, "null argument");
  return cudaEventQuery(h->out_done->e) == cudaSuccess ? 1 : 0;
}

int lms_handle_release(lms_ctx* c, lms_handle* h) {
  if (!c || !h) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  if (h->released) return fail(LMS_E_STATE, "double release");
  h->released = true;
  c->st.n_handles_live--;
  c->zombie.push_back(h);
  reap_zombies(c);
  return LMS_OK;
}

int lms_handle_info(lms_handle* h, int64_t* id, uint64_t* logical, uint64_t* wire, int* codec) {
  if (!h) return fail(LMS_E_INVALID, "null handle");
  if (!h->wire_known && cudaEventQuery(h->out_done->e) == cudaSuccess) h->wire = zvc_wire_bytes(h->host, h->host_bytes);
  if (id) *id = h->id;
  if (logical) *logical = h->logical;
  if (wire) *wire = h->wire;
  if (codec) *codec = h->codec;
  return LMS_OK;
}

int lms_handle_layout(lms_handle* h, int64_t* strides_out, int64_t* storage_elems) {
  if (!h) return fail(LMS_E_INVALID, "null handle");
  if (h->packed) {
    int64_t acc = 1;
    for (int k = h->ndim - 1; k >= 0; --k) {
      if (strides_out) strides_out[k] = acc;
      acc *= h->sizes[k];
    }
    if (storage_elems) *storage_elems = h->numel;
  } else {
    for (int k = 0; k < h->ndim; ++k)
      if (strides_out) strides_out[k] = h->strides[k];
    if (storage_elems) *storage_elems = h->span;
  }
  return LMS_OK;
}

static bool view_empty(int ndim, const int64_t* sizes) {
  for (int k = 0; k < ndim; ++k)
    if (sizes[k] == 0) return true;
  return false;
}

int lms_pack(lms_ctx* c, void* dst, const void* src, const int64_t* sizes, const int64_t* strides, int ndim,
             int elem_size, void* stream) {
  if (c && ndim >= 0 && ndim <= LMS_MAX_DIMS && view_empty(ndim, sizes)) return LMS_OK;
  if (!c || !dst || !src) return fail(LMS_E_INVALID, "null argument");
  if (ndim < 0 || ndim > LMS_MAX_DIMS) return fail(LMS_E_INVALID, "ndim out of range");
  return launch_layout<true>(c, static_cast<char*>(dst), static_cast<const char*>(src), ndim, sizes, strides,
                             elem_size, static_cast<cudaStream_t>(stream), kMemUnknown);
}

int lms_unpack(lms_ctx* c, void* dst, const void* src, const int64_t* sizes, const int64_t* strides, int ndim,
               int elem_size, void* stream) {
  if (c && ndim >= 0 && ndim <= LMS_MAX_DIMS && view_empty(ndim, sizes)) return LMS_OK;
  if (!c || !dst || !src) return fail(LMS_E_INVALID, "null argument");
  if (ndim < 0 || ndim > LMS_MAX_DIMS) return fail(LMS_E_INVALID, "ndim out of range");
  return launch_layout<false>(c, static_cast<char*>(dst), static_cast<const char*>(src), ndim, sizes, strides,
                              elem_size, static_cast<cudaStream_t>(stream), kMemUnknown);
}

size_t lms_zvc_bound(size_t nwords) { return zvc_bound(nwords); }

int lms_zvc_encode(lms_ctx* c, const void* src, size_t nwords, void* dst, int exponents, void* stream) {
  if (!c || (!src && nwords) || !dst) return fail(LMS_E_INVALID, "null argument");
  if (reinterpret_cast<uintptr_t>(src) % 16 || reinterpret_cast<uintptr_t>(dst) % 16)
    return fail(LMS_E_INVALID, "zvc buffers must be 16-byte aligned");
  std::lock_guard<std::mutex> g(c->mu);
  return launch_zvc_encode(c, static_cast<const uint32_t*>(src), nwords, static_cast<char*>(dst),
                           static_cast<cudaStream_t>(stream), is_host_ptr(dst), exponents != 0);
}

int lms_zvc_decode(lms_ctx* c, const void* enc, size_t nwords, void* dst, void* stream) {
  if (!c || !enc || (!dst && nwords)) return fail(LMS_E_INVALID, "null argument");
  if (nwords == 0) return LMS_OK;
  return launch_zvc_decode(c, static_cast<const char*>(enc), nwords, static_cast<uint32_t*>(dst),
                           static_cast<cudaStream_t>(stream), is_host_ptr(enc));
}

int lms_sim_op(lms_ctx* c, void* const* outs, const uint64_t* out_bytes, const uint32_t* out_tags, int n_out,
               const void* const* ins, const uint64_t* in_bytes, const uint32_t* in_tags, int n_in,
               uint64_t spin_ns, uint32_t* errors, void* stream) {
  if (!c || !errors || n_in < 0 || n_out < 0 || (n_in && (!ins || !in_bytes || !in_tags)) ||
      (n_out && (!outs || !out_bytes || !out_tags)))
    return fail(LMS_E_INVALID, "lms_sim_op: null argument");
  uint64_t total = 0;
  for (int k = 0; k < n_in; ++k) total += in_bytes[k];
  for (int k = 0; k < n_out; ++k) total += out_bytes[k];
  // ops with more operands than one launch carries run as several launches
  int i0 = 0, o0 = 0;
  do {
    SimArgs a{};
    a.n_in = std::min(n_in - i0, kSimMaxArgs);
    a.n_out = std::min(n_out - o0, kSimMaxArgs);
    for (int k = 0; k < a.n_in; ++k) {
      a.in[k] = ins[i0 + k];
      a.in_bytes[k] = in_bytes[i0 + k];
      a.in_tag[k] = in_tags[i0 + k];
    }
    for (int k = 0; k < a.n_out; ++k) {
      a.out[k] = outs[o0 + k];
      a.out_bytes[k] = out_bytes[o0 + k];
      a.out_tag[k] = out_tags[o0 + k];
    }
    i0 += a.n_in;
    o0 += a.n_out;
    const bool last = i0 >= n_in && o0 >= n_out;
    const int grid = sm_grid(c, int64_t(total / 16 + 1), 256 * 4);
    sim_op_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, last ? spin_ns : 0, errors);
    c->st.kernel_launches++;
    CK(cudaGetLastError());
  } while (i0 < n_in || o0 < n_out);
  return LMS_OK;
}

int lms_zvc_encoded_size(const void* enc_host, size_t* out) {
  if (!enc_host || !out) return fail(LMS_E_INVALID, "null argument");
  const ZvcHeader* h = static_cast<const ZvcHeader*>(enc_host);
  if (h->magic != kZvcMagic) return fail(LMS_E_INVALID, "not a ZVC stream");
  *out = zvc_wire_bytes(static_cast<const char*>(enc_host), 0);
  return LMS_OK;
}

int lms_stats(lms_ctx* c, lms_stats_t* out) {
  if (!c || !out) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  reap_deferred(c, false);
  account_zvc(c);
  lms_stats_t s = c->st;
  s.device_in_use = dev_in_use(c);
  s.device_peak = c->alloc_peak;
  s.device_reserved = c->vmm ? c->vmm->va_bytes() : 0;
  s.device_limit = c->limit;
  s.device_cached = c->vmm ? c->vmm->mapped_bytes() - std::min(c->vmm->mapped_bytes(), c->alloc_bytes) : 0;
  s.device_mapped = c->vmm ? c->vmm->mapped_bytes() : 0;
  s.device_mapped_peak = c->mapped_peak;
  s.n_map = c->vmm ? c->vmm->n_map() : 0;
  s.n_unmap = c->vmm ? c->vmm->n_unmap() : 0;
  s.n_reclaims = c->vmm ? c->vmm->n_moves() : 0;
  s.n_device_syncs = c->n_device_syncs;
  s.pool_driver_ms = c->vmm ? c->vmm->driver_ms() : 0;
  s.unmap_ms = c->vmm ? c->vmm->unmap_ms() : 0;
  s.map_ms = c->vmm ? c->vmm->map_ms() : 0;
  s.access_ms = c->vmm ? c->vmm->access_ms() : 0;
  s.device_deferred_bytes = c->deferred_bytes;
  s.host_in_use = c->host_used;
  s.host_peak = c->host_peak;
  s.host_reserved = c->host_reserved;
  s.numa_node = c->numa_node;
  s.n_host_chunks_on_node = c->chunks_on_node;
  double d2h = 0, h2d = 0;
  for (auto& r : c->recs) {
    if (cudaEventQuery(r.end) != cudaSuccess) continue;
    float ms = 0;
    cudaEventElapsedTime(&ms, r.start, r.end);
    (r.direction == 0 ? d2h : h2d) += ms;
  }
  s.d2h_busy_ms = d2h;
  s.h2d_busy_ms = h2d;
  double stall = 0;
  for (auto& w : c->waits) {
    const XferRec& r = c->recs[w.second];
    if (cudaEventQuery(w.first) != cudaSuccess || cudaEventQuery(r.end) != cudaSuccess) continue;
    float ms = 0;
    cudaEventElapsedTime(&ms, w.first, r.end);
    if (ms > 0) stall += ms;
  }
  s.swap_wait_ms = stall;
  *out = s;
  return LMS_OK;
}

int lms_live_blocks(lms_ctx* c, uint64_t* sizes, size_t cap, size_t* n) {
  if (!c || !n) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  std::vector<uint64_t> v;
  if (c->vmm) {
    c->vmm->for_each_live([&](uint64_t s) { v.push_back(s); });
  }
  std::sort(v.begin(), v.end(), std::greater<uint64_t>());
  size_t k = std::min(cap, v.size());
  if (sizes)
    for (size_t i = 0; i < k; ++i) sizes[i] = v[i];
  *n = v.size();
  return LMS_OK;
}

int lms_trace(lms_ctx* c, lms_xfer_record_t* out, size_t cap, size_t* n) {
  if (!c || !n) return fail(LMS_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  size_t k = 0;
  for (auto& r : c->recs) {
    if (k >= cap) break;
    if (cudaEventQuery(r.end) != cudaSuccess) continue;
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, c->epoch, r.start);
    cudaEventElapsedTime(&b, c->epoch, r.end);
    if (out) out[k] = {r.handle_id, r.direction, r.codec, r.logical, r.wire, a, b};
    ++k;
  }
  *n = k;
  return LMS_OK;
}

int lms_trace_clear(lms_ctx* c) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  cudaStreamSynchronize(c->d2h);
  cudaStreamSynchronize(c->h2d);
  for (auto& r : c->recs) {
    c->events.put(r.start, true);
    c->events.put(r.end, true);
  }
  c->recs.clear();
  c->trace_gen++;
  for (auto& w : c->waits) c->events.put(w.first, true);
  c->waits.clear();
  cudaEventRecord(c->epoch, c->d2h);
  c->st.d2h_logical_bytes = c->st.d2h_wire_bytes = 0;
  c->st.h2d_logical_bytes = c->st.h2d_wire_bytes = 0;
  c->st.n_swap_out = c->st.n_swap_in = 0;
  c->st.kernel_launches = 0;
  return LMS_OK;
}

int lms_trim(lms_ctx* c, size_t min_zombies, size_t* n) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  size_t z = c->vmm ? c->vmm->zombies() : 0;
  if (z < std::max<size_t>(min_zombies, 1)) z = 0;
  if (z) c->vmm->trim();
  if (n) *n = z;
  return LMS_OK;
}

int lms_synchronize(lms_ctx* c) {
  if (!c) return fail(LMS_E_INVALID, "null ctx");
  CK(cudaStreamSynchronize(c->d2h));
  CK(cudaStreamSynchronize(c->h2d));
  std::lock_guard<std::mutex> g(c->mu);
  reap_deferred(c, false);
  reap_zombies(c);
  if (c->vmm) c->vmm->trim();
  return LMS_OK;
}

// PyTorch CUDAPluggableAllocator hooks.  The pluggable ABI has no error
// channel, so an exhausted budget is reported by throwing: PyTorch's Python
// boundary turns it into a RuntimeError whose text starts with "LMS_OOM".
void* lms_alloc(size_t size, int device, void* stream) {
  lms_ctx* c = g_global;
  if (!c) throw std::runtime_error("LMS: allocator hook called before lms_set_global");
  (void)device;
  void* p = nullptr;
  int rc;
  {
    std::lock_guard<std::mutex> g(c->mu);
    rc = dev_alloc_locked(c, size, stream, &p);
  }
  if (rc != LMS_OK) throw OomError(g_err);
  return p;
}

void lms_free(void* ptr, size_t size, int device, void* stream) {
  (void)size;
  (void)device;
  lms_ctx* c = g_global;
  if (!c) return;
  std::lock_guard<std::mutex> g(c->mu);
  dev_free_locked(c, ptr, stream);
}

}  // extern "C"
