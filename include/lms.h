/*
 * liblms.so — C ABI of the B200 executor runtime for TFLMS-style swapping.
 *
 * The reference package (swapgraph) has no FFI: its executor and its
 * transfer/memory model are Python functions.  This header is the boundary
 * that replaces them; every entry point names the reference behaviour it
 * implements:
 *
 *   device pool      <- residency/refcount model, sim.py:116-124, :193-211,
 *                       :356-401 (alloc at op start, free at refcount 0 AND
 *                       after outbound transfers, sim.py:205-211, :379-386);
 *                       capacity/OOM, sim.py:49, :471
 *   host pool        <- host residency of swapped tensors, sim.py:193-199
 *   swap_out/in      <- swap node semantics: identity on values
 *                       (interp.py:168-170) realised as D2H/H2D transfers on
 *                       per-direction channels (sim.py:284-322); the swap-in
 *                       is gated by its control edge (rewriter.py:455-477,
 *                       control.py:158-169)
 *   stats / trace    <- SimReport / TraceEvent schema, sim.py:74-113
 *
 * Conventions: functions return 0 on success and a negative LMS_E* code on
 * failure; lms_last_error() gives the message (thread-local).  Nothing
 * throws across the ABI.  Pointers are plain device / host pointers,
 * streams and events are CUDA runtime handles passed as void*.
 * The four allocator hooks at the bottom have exactly the signatures of
 * PyTorch's CUDAPluggableAllocator (torch/csrc/cuda/CUDAPluggableAllocator.h:
 * alloc_fn(size_t, int, cudaStream_t), free_fn(void*, size_t, int,
 * cudaStream_t)).
 */
#ifndef LMS_H_
#define LMS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMS_MAX_DIMS 8

enum {
  LMS_OK = 0,
  LMS_E_INVALID = -1,   /* bad argument (ValueError in the Python wrapper) */
  LMS_E_OOM = -2,       /* device budget exceeded (SimReport.oom analogue) */
  LMS_E_HOST_OOM = -3,  /* pinned host pool cannot grow */
  LMS_E_CUDA = -4,      /* CUDA runtime error; message has the details */
  LMS_E_STATE = -5      /* call out of order (e.g. swap_in of a released handle) */
};

/* Transfer codecs for swap-out.  RAW_CE moves the tensor's storage span with
 * the copy engine (packing first only when the view is not dense).  RAW_SM
 * moves it with an SM kernel writing straight into mapped pinned memory
 * (fused pack for strided views).  ZVC is a lossless tile codec over 32-bit
 * words: one SM kernel pass writes, per 16 KiB tile, either the words or a
 * zero bitmask plus the nonzero words straight into pinned memory, and the
 * swap-in decodes straight out of it (only encoded bytes cross the link).
 * ZX is ZVC plus exponent planes: a tile may also store each word's low 24
 * bits and its top byte coded in the tile's narrow exponent band (k bits +
 * a sign bit unless all signs agree) — lossless, for dense fp32 tensors. */
enum { LMS_CODEC_RAW_CE = 0, LMS_CODEC_RAW_SM = 1, LMS_CODEC_ZVC = 2, LMS_CODEC_ZX = 3 };

typedef struct lms_ctx lms_ctx;
typedef struct lms_handle lms_handle;

typedef struct {
  int device;                 /* CUDA ordinal */
  size_t device_reserve;      /* bytes reserved for the device arena (0 = none yet) */
  size_t device_limit;        /* enforced budget in bytes (0 = arena size) */
  size_t host_reserve;        /* pinned bytes to pre-allocate */
  size_t host_chunk;          /* growth granularity of the pinned pool */
  int overlap_transfers;      /* 1: separate D2H/H2D streams (sim.py:287-290) */
  int timing;                 /* 1: record per-transfer timing events */
  int sm_ctas;                /* CTAs for SM-driven transfer/codec kernels (0 = auto) */
  size_t host_limit;          /* cap on pinned host bytes (0 = none); swap-outs past it fail
                                 with LMS_E_HOST_OOM instead of pinning the host into swap */
} lms_config_t;

typedef struct {
  uint64_t device_in_use, device_peak;         /* live block bytes (the model's residency) */
  uint64_t device_reserved, device_limit;      /* VA reserved; physical budget */
  uint64_t device_cached, device_deferred_bytes;   /* mapped free blocks; frees awaiting swap-outs */
  uint64_t device_mapped, device_mapped_peak;  /* physical pages actually backing blocks */
  uint64_t n_map, n_unmap, n_reclaims, n_device_syncs;
  uint64_t host_in_use, host_peak, host_reserved;
  uint64_t n_alloc, n_free, n_oom, n_deferred_frees, n_cross_stream_waits;
  uint64_t n_swap_out, n_swap_in, n_handles_live;
  uint64_t d2h_logical_bytes, d2h_wire_bytes;   /* tensor bytes vs bytes on PCIe */
  uint64_t h2d_logical_bytes, h2d_wire_bytes;
  uint64_t kernel_launches;                     /* our sm_100a kernels */
  double d2h_busy_ms, h2d_busy_ms;              /* sum of transfer spans (timing=1) */
  double swap_wait_ms;  /* consumer stalls on swap-ins (timing=1): transfer_wait_total */
  double pool_driver_ms;   /* host time in cuMemMap / cuMemSetAccess / cuMemUnmap */
  double alloc_wait_ms;    /* host time allocations spent waiting for swap-out copies */
  double host_grow_ms;     /* host time pinning new host-pool chunks (cudaHostAlloc) */
  uint64_t n_host_grow;    /* pinned chunks added */
  uint64_t n_scratch_grow; /* always 0 (the one-pass ZVC v3 codec has no scratch); kept for the ABI */
  double unmap_ms, map_ms, access_ms;  /* pool_driver_ms split by driver call */
  int64_t numa_node;              /* the GPU's NUMA node pinned chunks are placed on (-1: none) */
  uint64_t n_host_chunks_on_node; /* pinned chunks whose pages landed on that node */
} lms_stats_t;

/* one measured transfer, in the TraceEvent vocabulary (sim.py:74-81) */
typedef struct {
  int64_t handle_id;
  int direction;        /* 0 = D2H (swap-out), 1 = H2D (swap-in) */
  int codec;
  uint64_t logical_bytes, wire_bytes;
  double start_ms, end_ms;   /* relative to the context epoch */
} lms_xfer_record_t;

const char* lms_last_error(void);
const char* lms_version(void);

/* ---- context ------------------------------------------------------------ */
int lms_default_config(lms_config_t* cfg);
int lms_create(const lms_config_t* cfg, lms_ctx** out);
int lms_destroy(lms_ctx* ctx);
/* The context the allocator hooks below use (one per process / device). */
int lms_set_global(lms_ctx* ctx);
lms_ctx* lms_get_global(void);
/* Stream that owns freed blocks for immediate reuse (torch's compute stream). */
int lms_set_home_stream(lms_ctx* ctx, void* stream);
int lms_set_limit(lms_ctx* ctx, size_t limit);
int lms_reset_peaks(lms_ctx* ctx);
int lms_get_streams(lms_ctx* ctx, void** d2h, void** h2d);
/* Tuning: CTAs per zero-copy kernel launch (0 = keep); whether the ZVC
 * kernels move chunks with bulk async copies (1, TMA path) or with per-thread
 * 16 B loads/stores (0); whether pack/unpack of rows layouts in HBM go
 * through tensor maps (1, cp.async.bulk.tensor) or the SIMT kernels (0).
 * -1 keeps the current setting. */
int lms_set_tuning(lms_ctx* ctx, int zc_ctas, int use_bulk, int use_tma_pack);

/* ---- device pool (replaces the simulator's residency model) ------------- */
int lms_dev_alloc(lms_ctx* ctx, size_t size, void* stream, void** out);
int lms_dev_free(lms_ctx* ctx, void* ptr, void* stream);
/* keep the block containing ptr from reuse until the work now enqueued on
 * `stream` completes (a pending outbound transfer), like sim.py:205-211
 * "free after transfers done" */
int lms_dev_hold_until(lms_ctx* ctx, const void* ptr, void* stream);
/* the block containing ptr is also used on `stream` (PyTorch's recordStream):
 * when it is freed, its reuse waits for the work then enqueued on `stream` */
int lms_dev_record_stream(lms_ctx* ctx, const void* ptr, void* stream);
/* storage layout the swap-in restores by default: strides (elements) and the
 * number of storage elements to allocate */
int lms_handle_layout(lms_handle* h, int64_t* strides_out, int64_t* storage_elems);

/* ---- static step plan ------------------------------------------------------ */
/* A training step allocates the same sizes in the same order every
 * iteration.  RECORD logs one step's allocations (size, alloc/free events);
 * lms_plan_end then places them once inside one contiguous region (greedy,
 * step_plan.h).  REPLAY serves each later step's allocations from the
 * recorded offsets: no fragmentation, no page moves; a step that allocates
 * differently falls back to the dynamic pool from the first mismatch on.
 * Residency intervals are the reference's model, sim.py:116-124, :193-211. */
/* REFINE replays like REPLAY and also observes when each planned block's
 * swap-out copy finished; lms_plan_end then re-places the step with those
 * (replay-speed) lifetimes and adopts the result if it fits the region. */
enum { LMS_PLAN_OFF = 0, LMS_PLAN_RECORD = 1, LMS_PLAN_REPLAY = 2, LMS_PLAN_REFINE = 3 };
int lms_plan_begin(lms_ctx* ctx, int mode);
/* ends the step; after RECORD it solves the placement and reserves the
 * region (LMS_E_OOM if the region does not fit the budget: no plan) */
int lms_plan_end(lms_ctx* ctx);
/* drops the plan and returns its region to the pool (no planned block may be live) */
int lms_plan_reset(lms_ctx* ctx);
typedef struct {
  int ready;
  uint64_t region_bytes, lower_bound_bytes;   /* placement vs max live bytes */
  uint64_t n_items, n_planned;
  uint64_t hits, dynamic, diverged_steps;
  uint64_t solved_bytes;   /* region the last solve needed (also when it did not fit) */
  uint64_t room_bytes;     /* budget left for a region next to the live set */
  double alpha;            /* lifetime ends used: 1 = physical releases (after swap-out copies),
                              0 = the owners' frees (step_plan.h plan_place_fit) */
  uint64_t refinements;    /* REFINE steps whose re-placement was adopted */
} lms_plan_info_t;
int lms_plan_info(lms_ctx* ctx, lms_plan_info_t* out);
/* the recording step's event clock so far (-1 outside RECORD): lets a caller
 * place its own host events (e.g. a control op firing) on the items' clock */
int lms_plan_clock(lms_ctx* ctx, int64_t* out);
/* the recorded step (after lms_plan_end of a RECORD step): up to `cap` items */
int lms_plan_items(lms_ctx* ctx, uint64_t* sizes, int64_t* t_alloc, int64_t* t_free, int64_t* t_free_logical,
                   size_t cap, size_t* n);
/* the placement on its own (host only): n items with sizes and alloc/free
 * events (free < 0: not planned) -> offsets; returns region size via *region */
int lms_plan_solve(const uint64_t* sizes, const int64_t* t_alloc, const int64_t* t_free, size_t n,
                   uint64_t* offsets, uint64_t* region);

/* ---- host pool ------------------------------------------------------------ */
int lms_host_alloc(lms_ctx* ctx, size_t size, void** out);
int lms_host_free(lms_ctx* ctx, void* ptr);
/* grow the pinned pool to at least `total` reserved bytes now (cudaHostAlloc is
 * slow and may stall the device: keep it out of timed steps) */
int lms_host_reserve(lms_ctx* ctx, size_t total);

/* ---- swap engine ------------------------------------------------------------ */
/* Swap-out: the D2H channel waits for the work already enqueued on
 * `producer_stream`, then moves the tensor (sizes/strides in elements) to
 * pinned memory with `codec`.  The source block is held until the transfer
 * completes, so freeing it right away is safe. */
int lms_swap_out(lms_ctx* ctx, const void* src, const int64_t* sizes, const int64_t* strides,
                 int ndim, int elem_size, void* producer_stream, int codec, lms_handle** out);
/* Swap-in: the H2D channel waits for the work already enqueued on
 * `trigger_stream` (the control op's completion point) and for the swap-out,
 * then restores the values into `dst` (layout `dst_strides`, or contiguous
 * when NULL). */
int lms_swap_in(lms_ctx* ctx, lms_handle* h, void* dst, const int64_t* dst_strides,
                void* trigger_stream);
/* Make `consumer_stream` wait until the last swap-in of `h` has landed. */
int lms_swap_wait(lms_ctx* ctx, lms_handle* h, void* consumer_stream);
/* Host-side query: 1 if the swap-out finished, 0 if still in flight. */
int lms_swap_out_done(lms_ctx* ctx, lms_handle* h);
/* Release the host copy (deferred until pending H2D reads finish). */
int lms_handle_release(lms_ctx* ctx, lms_handle* h);
int lms_handle_info(lms_handle* h, int64_t* id, uint64_t* logical_bytes, uint64_t* wire_bytes,
                    int* codec);

/* ---- staging kernels (sm_100a), usable on their own ------------------------ */
/* dst (contiguous) <- src (strided view) */
int lms_pack(lms_ctx* ctx, void* dst, const void* src, const int64_t* sizes,
             const int64_t* strides, int ndim, int elem_size, void* stream);
/* dst (strided view) <- src (contiguous) */
int lms_unpack(lms_ctx* ctx, void* dst, const void* src, const int64_t* sizes,
               const int64_t* strides, int ndim, int elem_size, void* stream);
/* ZVC / ZX codec over `nwords` 32-bit words (exponents != 0: ZX tile forms
 * allowed); encode writes to any device-visible buffer (pinned host included)
 * of at least lms_zvc_bound(nwords) bytes, one pass over the source, each
 * tile into its own fixed 16 KiB slot.  Stream format: kernels.cuh (ZVC v3). */
size_t lms_zvc_bound(size_t nwords);
int lms_zvc_encode(lms_ctx* ctx, const void* src, size_t nwords, void* dst, int exponents, void* stream);
int lms_zvc_decode(lms_ctx* ctx, const void* enc, size_t nwords, void* dst, void* stream);
/* bytes an encoded stream put on the wire (header + tile table + chunks);
 * the stream must be host-readable */
int lms_zvc_encoded_size(const void* enc_host, size_t* out);

/* ---- measured simulation (replaces sim.py:139-476's modelled op) ----------- */
/* One graph op of a replayed schedule (the GPU-measured `simulate`): checks
 * each input against the word pattern of its origin tensor tag (mismatching
 * words are added to *errors, a device counter), fills each output with its
 * own tag's pattern, and lasts at least spin_ns (the node's cost_hint,
 * sim.py:350-352).  Ops with more than 8 inputs/outputs take several launches. */
int lms_sim_op(lms_ctx* ctx, void* const* outs, const uint64_t* out_bytes, const uint32_t* out_tags, int n_out,
               const void* const* ins, const uint64_t* in_bytes, const uint32_t* in_tags, int n_in,
               uint64_t spin_ns, uint32_t* errors, void* stream);

/* ---- stats / trace -------------------------------------------------------- */
/* sizes of live device blocks, largest first (diagnostics); *n = total count */
int lms_live_blocks(lms_ctx* ctx, uint64_t* sizes, size_t cap, size_t* n);
int lms_stats(lms_ctx* ctx, lms_stats_t* out);
/* copies up to `cap` finished transfer records; returns count via *n */
int lms_trace(lms_ctx* ctx, lms_xfer_record_t* out, size_t cap, size_t* n);
int lms_trace_clear(lms_ctx* ctx);
int lms_synchronize(lms_ctx* ctx);
/* Unmap the stale VA aliases page moves leave behind (each cuMemUnmap waits
 * for the device to drain, so this belongs at a step boundary) once there are
 * at least `min_zombies` of them; the number unmapped via *n (may be NULL). */
int lms_trim(lms_ctx* ctx, size_t min_zombies, size_t* n);

/* ---- PyTorch CUDAPluggableAllocator hooks (use the global context) -------- */
void* lms_alloc(size_t size, int device, void* stream);
void lms_free(void* ptr, size_t size, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LMS_H_ */
