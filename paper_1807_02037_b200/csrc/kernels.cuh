// sm_100a staging and transfer kernels for the swap engine.
//
// Everything here is bandwidth work (HBM on one side, PCIe on the other for
// the zero-copy variants), so the design rules are: 128-bit accesses where
// alignment allows, several independent loads in flight per thread, grids
// sized to the SM count, and shared-memory tiles only where a layout change
// (transpose) would otherwise make one side uncoalesced.
//
//   pack/unpack   strided view <-> contiguous staging (rows / transpose /
//                 generic paths)
//   copy16        device<->pinned-host streaming copy driven by SMs
//                 (zero-copy: the "kernel" transfer engine)
//   zvc_*         lossless tile codec of 32-bit words (zero masks and
//                 exponent planes), one pass straight into pinned memory,
//                 decoded straight out of it
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace lms {

constexpr int kMaxDims = 8;

struct Strided {
  int ndim;
  int64_t sizes[kMaxDims];
  int64_t strides[kMaxDims];  // elements
};

// -------------------------------------------------------------------------
// helpers

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// element offset of logical linear index `i` under `d`, skipping the dims in
// [skip_lo, ndim) (they are handled by the caller)
__device__ __forceinline__ int64_t outer_offset(const Strided& d, int64_t i, int upto) {
  int64_t off = 0;
#pragma unroll
  for (int k = kMaxDims - 1; k >= 0; --k) {
    if (k < upto) {
      int64_t s = d.sizes[k];
      int64_t q = i / s;
      off += (i - q * s) * d.strides[k];
      i = q;
    }
  }
  return off;
}

template <int E> struct Word;
template <> struct Word<1> { using T = uint8_t; };
template <> struct Word<2> { using T = uint16_t; };
template <> struct Word<4> { using T = uint32_t; };
template <> struct Word<8> { using T = uint64_t; };

// -------------------------------------------------------------------------
// pack / unpack, "rows" path: the strided side's last dim is unit-stride, so
// each logical row of R elements is a contiguous run.  kVec: rows are 16B
// multiples and 16B aligned on both sides -> uint4 copies.
// PACK=true: dst contiguous, src strided.  PACK=false: the reverse.

template <bool PACK, bool kVec, int E>
__global__ void __launch_bounds__(256) rows_kernel(char* __restrict__ dst, const char* __restrict__ src,
                                                   Strided d, int64_t rows, int64_t row_len) {
  using T = typename Word<E>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    int64_t soff = outer_offset(d, r, d.ndim - 1) * E;  // strided-side byte offset of row r
    int64_t coff = r * row_len * E;                     // contiguous-side byte offset
    const char* s = PACK ? src + soff : src + coff;
    char* t = PACK ? dst + coff : dst + soff;
    if (kVec) {
      int64_t n16 = row_len * E / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* t4 = reinterpret_cast<uint4*>(t);
      int64_t j = lane;
      for (; j + 96 < n16; j += 128) {  // 4 loads in flight per lane
        uint4 a = ld_stream(s4 + j), b = ld_stream(s4 + j + 32);
        uint4 c = ld_stream(s4 + j + 64), e = ld_stream(s4 + j + 96);
        t4[j] = a; t4[j + 32] = b; t4[j + 64] = c; t4[j + 96] = e;
      }
      for (; j < n16; j += 32) t4[j] = ld_stream(s4 + j);
    } else {
      const T* sw = reinterpret_cast<const T*>(s);
      T* tw = reinterpret_cast<T*>(t);
      for (int64_t j = lane; j < row_len; j += 32) tw[j] = sw[j];
    }
  }
}

// -------------------------------------------------------------------------
// transpose path: the strided side has a unit-stride dim `cd` (not the last
// one) and its last dim is strided.  A 32x32 tile over (cd, last) is read
// coalesced along cd and written coalesced along last through shared memory.
// Index math is per tile (64-bit tile bases, one pass over the batch dims);
// per element only 32-bit in-tile offsets (host checks 32*stride < 2^31).

template <bool PACK, int E>
__global__ void __launch_bounds__(256) transpose_kernel(char* __restrict__ dst, const char* __restrict__ src,
                                                        Strided d, int cd, int64_t batches) {
  using T = typename Word<E>::T;
  __shared__ T tile[32][33];
  const int last = d.ndim - 1;
  const int64_t nA = d.sizes[cd], nB = d.sizes[last];
  const int64_t tilesA = (nA + 31) / 32, tilesB = (nB + 31) / 32;
  const int64_t ntiles = batches * tilesA * tilesB;
  // row-major strides of the contiguous side
  int64_t cstride[kMaxDims];
  {
    int64_t acc = 1;
#pragma unroll
    for (int k = kMaxDims - 1; k >= 0; --k) {
      if (k < d.ndim) {
        cstride[k] = acc;
        acc *= d.sizes[k];
      }
    }
  }
  const uint32_t sA = uint32_t(d.strides[cd]), sB = uint32_t(d.strides[last]);  // strided side
  const uint32_t cA = uint32_t(cstride[cd]);                                      // contiguous side (cB = 1)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const T* sw = reinterpret_cast<const T*>(src);
  T* dw = reinterpret_cast<T*>(dst);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t / (tilesA * tilesB);
    const int64_t rem = t - b * tilesA * tilesB;
    const int64_t ta = rem / tilesB;
    const int64_t a0 = ta * 32, b0 = (rem - ta * tilesB) * 32;
    // batch index -> offsets over the dims other than cd and last
    int64_t soff = 0, coff = 0, bi = b;
    for (int k = last - 1; k >= 0; --k) {
      if (k == cd) continue;
      const int64_t s = d.sizes[k];
      const int64_t q = bi / s;
      const int64_t x = bi - q * s;
      soff += x * d.strides[k];
      coff += x * cstride[k];
      bi = q;
    }
    const int ra = int(nA - a0 < 32 ? nA - a0 : 32), rb = int(nB - b0 < 32 ? nB - b0 : 32);
    const int64_t s_org = soff + a0 * d.strides[cd] + b0 * d.strides[last];  // strided-side tile origin
    const int64_t c_org = coff + a0 * cstride[cd] + b0;                       // contiguous-side tile origin
    T v[4];
    if (PACK) {
      const T* sp = sw + s_org;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = ty + 8 * k;  // b (last) index; tx runs along the unit-stride a
        v[k] = (tx < ra && j < rb) ? sp[uint32_t(tx) * sA + uint32_t(j) * sB] : T(0);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) tile[ty + 8 * k][tx] = v[k];
      __syncthreads();
      T* cp = dw + c_org;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = ty + 8 * k;  // a index; tx runs along the contiguous b
        if (j < ra && tx < rb) cp[uint32_t(j) * cA + tx] = tile[tx][j];
      }
    } else {
      const T* cp = sw + c_org;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = ty + 8 * k;  // a index; tx runs along the contiguous b
        v[k] = (j < ra && tx < rb) ? cp[uint32_t(j) * cA + tx] : T(0);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) tile[ty + 8 * k][tx] = v[k];
      __syncthreads();
      T* sp = dw + s_org;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = ty + 8 * k;  // b index; tx runs along the unit-stride a
        if (tx < ra && j < rb) sp[uint32_t(tx) * sA + uint32_t(j) * sB] = tile[tx][j];
      }
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------------------
// generic path: any strides (including 0 and negative), one element per step

template <bool PACK, int E>
__global__ void __launch_bounds__(256) generic_kernel(char* __restrict__ dst, const char* __restrict__ src,
                                                      Strided d, int64_t numel) {
  using T = typename Word<E>::T;
  const T* sw = reinterpret_cast<const T*>(src);
  T* dw = reinterpret_cast<T*>(dst);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < numel;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t so = outer_offset(d, i, d.ndim);
    if (PACK) dw[i] = sw[so]; else dw[so] = sw[i];
  }
}

// -------------------------------------------------------------------------
// copy16: streaming copy between any two device-visible buffers (HBM or
// mapped pinned host).  Both pointers 16B aligned; n16 16-byte words.
// Each thread keeps 4 independent 16B loads in flight so a few dozen CTAs
// cover PCIe latency without taking SMs away from the compute stream.

__global__ void __launch_bounds__(512) copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                     int64_t n16) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  int64_t i = tid;
  for (; i + 3 * nth < n16; i += 4 * nth) {
    uint4 a = ld_stream(src + i), b = ld_stream(src + i + nth);
    uint4 c = ld_stream(src + i + 2 * nth), e = ld_stream(src + i + 3 * nth);
    st_stream(dst + i, a); st_stream(dst + i + nth, b);
    st_stream(dst + i + 2 * nth, c); st_stream(dst + i + 3 * nth, e);
  }
  for (; i < n16; i += nth) st_stream(dst + i, ld_stream(src + i));
}

__global__ void copy_tail_kernel(char* __restrict__ dst, const char* __restrict__ src, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// -------------------------------------------------------------------------
// Bulk asynchronous copies (the 1-D TMA path: cp.async.bulk, SASS UBLKCP)
// and mbarriers.  Used by the ZVC kernels to move whole tile chunks between
// shared memory and global memory -- HBM or mapped pinned host memory.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "ZVC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra ZVC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global (HBM or mapped host) -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global (HBM or mapped host), tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N groups still reading their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// at most N groups not yet complete (writes performed)
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// generic-proxy shared-memory writes become visible to the async (bulk) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// -------------------------------------------------------------------------
// ZVC v3: lossless tile codec over 32-bit words, one pass over HBM.
//
// A swapped activation is encoded on its way out by SM kernels writing
// straight into mapped pinned memory, and decoded on its way in by SM
// kernels reading straight out of it, so only the encoded bytes cross the
// host link and no device staging buffer is taken from the budget.
//
// Every 4096-word (16 KiB) tile picks the smallest of four lossless forms:
//   RAW   the words
//   MASK  128-word bitmask (bit j of word s: word 32s+j is nonzero) + the
//         nonzero words                          (ReLU outputs: ~50 % zeros)
//   EXPD  every word split into its low 24 bits (3-byte plane) and its top
//         byte (sign + 7 high exponent bits), the top bytes coded as
//         (e7 - emin) in k bits plus a sign bit unless the tile's signs agree,
//         packed b = k + sign bits per word
//   EXPM  MASK's bitmask, then the nonzero words' low bytes (3 each) and their
//         codes packed b bits each
// (fp32 activations keep their exponents in a narrow band per tile: k is
// typically 3-4 of 7 bits, and ReLU outputs need no sign bit.)
//
// Stream layout (bytes; every region 16 B aligned):
//   [0, 64)                     header {magic "ZVC3", flags, nwords, ntiles, table_pos, data_pos}
//   [64, 64 + 8 ntiles)         per tile {u32 info, u32 bytes}: info = mode | k<<2 | signplane<<6 |
//                               sign<<7 | emin<<8 | n<<16 (n = words coded: tile words, or nnz)
//   [data_pos, ...)             tile t's chunk at data_pos + t * 16 KiB (fixed slots: no scan
//                               pass; only a chunk's own bytes are ever written or read)
// There is no global pass: a CTA encodes a tile from registers, builds the
// chunk in shared memory and stores it with one bulk copy.

constexpr int kZvcTileWords = 4096;
constexpr int kZvcMaskWords = kZvcTileWords / 32;                 // 128
constexpr uint32_t kZvcSlotBytes = kZvcTileWords * 4;             // 16 KiB
constexpr int kZvcBufBytes = kZvcSlotBytes + 512;                 // chunk buffer (+ scratch slack)
constexpr int kZvcSmemBytes = 2 * kZvcBufBytes;                   // double-buffered
constexpr int kZvcEncSmemBytes = kZvcSmemBytes + 2 * kZvcSlotBytes;  // + two prefetched input tiles
constexpr uint32_t kZvcMagic = 0x3343565Au;                       // "ZVC3"
enum { kZRaw = 0, kZMask = 1, kZExpD = 2, kZExpM = 3 };

struct ZvcHeader {
  uint32_t magic, flags;
  uint64_t nwords, ntiles, table_pos, data_pos;
  uint64_t pad[3];
};
static_assert(sizeof(ZvcHeader) == 64, "header is 64 bytes");

struct ZvcTile {
  uint32_t info, bytes;
};

__host__ __device__ inline uint64_t zvc_tiles(uint64_t nwords) {
  return (nwords + kZvcTileWords - 1) / kZvcTileWords;
}
__host__ __device__ inline uint64_t zvc_data_pos(uint64_t ntiles) { return 64 + (ntiles * 8 + 15) / 16 * 16; }
__host__ __device__ inline uint32_t zvc_pad16(uint64_t b) { return uint32_t((b + 15) / 16 * 16); }
// worst case: every chunk raw; the last tile's slot only needs its own words
__host__ __device__ inline uint64_t zvc_bound(uint64_t nwords) {
  const uint64_t t = zvc_tiles(nwords);
  if (t == 0) return 64;
  return zvc_data_pos(t) + (t - 1) * kZvcSlotBytes + zvc_pad16(4 * (nwords - (t - 1) * kZvcTileWords));
}

// exclusive scan of the 128 per-segment popcounts in seg[] (warp 0); seg[128] = total
__device__ __forceinline__ void zvc_seg_scan(uint32_t* seg, int lane) {
  uint32_t a = seg[lane * 4], b = seg[lane * 4 + 1], c = seg[lane * 4 + 2], e = seg[lane * 4 + 3];
  uint32_t s = a + b + c + e, x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const uint32_t ex = x - s;
  seg[lane * 4] = ex;
  seg[lane * 4 + 1] = ex + a;
  seg[lane * 4 + 2] = ex + a + b;
  seg[lane * 4 + 3] = ex + a + b + c;
  if (lane == 31) seg[kZvcMaskWords] = x;
}

__device__ __forceinline__ uint32_t zvc_nbits(uint32_t r) { return r ? 32u - __clz(r) : 0u; }

// exponent planes: word p's low 24 bits at byte 3p of `lo`, its code at bit p*b of `hi`
__device__ __forceinline__ void zvc_put_exp(unsigned char* lo, uint32_t* hi, uint32_t p, uint32_t w, uint32_t k,
                                            uint32_t sp, uint32_t emin) {
  lo[3 * p] = uint8_t(w);
  lo[3 * p + 1] = uint8_t(w >> 8);
  lo[3 * p + 2] = uint8_t(w >> 16);
  const uint32_t b = k + sp;
  if (b == 0) return;
  const uint32_t code = (((w >> 24) & 0x7Fu) - emin) | (sp ? (w >> 31) << k : 0u);
  const uint32_t o = p * b, q = o >> 5, sh = o & 31u;
  atomicOr(hi + q, code << sh);
  if (sh + b > 32) atomicOr(hi + q + 1, code >> (32 - sh));
}

__device__ __forceinline__ uint32_t zvc_get_exp(const unsigned char* lo, const uint32_t* hi, uint32_t p, uint32_t k,
                                                uint32_t sp, uint32_t sconst, uint32_t emin) {
  const uint32_t low = uint32_t(lo[3 * p]) | uint32_t(lo[3 * p + 1]) << 8 | uint32_t(lo[3 * p + 2]) << 16;
  const uint32_t b = k + sp;
  uint32_t code = 0;
  if (b) {
    const uint32_t o = p * b, q = o >> 5, sh = o & 31u;
    code = hi[q] >> sh;
    if (sh + b > 32) code |= hi[q + 1] << (32 - sh);
  }
  const uint32_t e7 = emin + (code & ((1u << k) - 1u));
  const uint32_t s = sp ? (code >> k) & 1u : sconst;
  return ((s << 7 | e7) << 24) | low;
}

// One pass: per tile, statistics of the 4096 words held in registers pick the
// form, the chunk is assembled in shared memory and leaves with one bulk
// store (TMA when use_bulk, else 16 B STG) into its fixed slot.  Double-
// buffered: tile k+1 is built while tile k's chunk is in flight.
template <bool kExp>
__global__ void __launch_bounds__(256, 3) zvc_encode_kernel(const uint32_t* __restrict__ src, uint64_t nwords,
                                                            char* __restrict__ out, int use_bulk) {
  constexpr int allow_exp = kExp;
  extern __shared__ __align__(128) unsigned char zsm[];
  __shared__ uint32_t red[8][9];
  const uint64_t ntiles = zvc_tiles(nwords);
  const uint64_t dpos = zvc_data_pos(ntiles);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ZvcHeader h{};
    h.magic = kZvcMagic;
    h.flags = uint32_t(allow_exp != 0);
    h.nwords = nwords;
    h.ntiles = ntiles;
    h.table_pos = 64;
    h.data_pos = dpos;
    const uint4* hs = reinterpret_cast<const uint4*>(&h);
    uint4* ho = reinterpret_cast<uint4*>(out);
    for (int k = 0; k < 4; ++k) ho[k] = hs[k];
  }
  ZvcTile* table = reinterpret_cast<ZvcTile*>(out + 64);
  char* data = out + dpos;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  // input tiles are prefetched one ahead by bulk copies (HBM -> shared) so a
  // CTA's loads overlap its previous tile's encode and store
  __shared__ __align__(8) uint64_t ibar[2];
  const bool pref = use_bulk && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const uint32_t* inbuf = reinterpret_cast<const uint32_t*>(zsm + kZvcSmemBytes);
  auto load_tile = [&](uint64_t tt, int b) {   // thread 0 only
    const uint64_t tb = tt * kZvcTileWords;
    const uint32_t nv = uint32_t(nwords - tb < kZvcTileWords ? nwords - tb : kZvcTileWords);
    const uint32_t bytes = (nv * 4) & ~15u;
    fence_proxy_async_smem();   // earlier generic reads of this buffer come first
    mbar_expect_tx(&ibar[b], bytes);
    if (bytes) bulk_g2s(zsm + kZvcSmemBytes + b * kZvcSlotBytes, src + tb, bytes, &ibar[b]);
  };
  if (pref) {
    if (threadIdx.x == 0) {
      mbar_init(&ibar[0], 1);
      mbar_init(&ibar[1], 1);
      fence_mbar_init();
      if (blockIdx.x < ntiles) load_tile(blockIdx.x, 0);
    }
    __syncthreads();
  }
  uint32_t iph0 = 0, iph1 = 0;
  int buf = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
    unsigned char* chunk = zsm + buf * kZvcBufBytes;
    uint32_t* cw = reinterpret_cast<uint32_t*>(chunk);
    if (use_bulk && threadIdx.x == 0) bulk_wait_read<1>();  // the store that last read this buffer
    __syncthreads();
    const uint64_t base = t * kZvcTileWords;
    const uint32_t nvalid = uint32_t(nwords - base < kZvcTileWords ? nwords - base : kZvcTileWords);
    uint32_t w16[16];
    if (pref) {
      if (threadIdx.x == 0 && t + gridDim.x < ntiles) load_tile(t + gridDim.x, buf ^ 1);
      if (buf == 0) {
        mbar_wait(&ibar[0], iph0);
        iph0 ^= 1;
      } else {
        mbar_wait(&ibar[1], iph1);
        iph1 ^= 1;
      }
      const uint32_t* win = inbuf + buf * kZvcTileWords;
      const uint32_t nbulk = (nvalid * 4 & ~15u) / 4;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t j = r * 256 + threadIdx.x;
        w16[r] = j < nbulk ? win[j] : (j < nvalid ? __ldg(src + base + j) : 0u);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint64_t i = base + r * 256 + threadIdx.x;
        w16[r] = i < nwords ? __ldg(src + i) : 0u;
      }
    }
    // per-tile statistics: nonzeros, and the top-byte ranges over all / nonzero
    // words.  Zero words (and the zero padding past nvalid) have top byte 0, so
    // the maximum and the sign OR over all words equal those over the nonzero
    // ones; the nonzero words' sign AND is "no nonzero positive word"; only the
    // all-words minimum and sign AND need the valid-word test (partial tiles).
    uint32_t nnz = 0, mn_a = 127, mx = 0, orv = 0, andv = ~0u, mn_z = 127, posnz = 0;
    auto tile_stats = [&](auto full) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t v = w16[r];
        nnz += v != 0;
        if (kExp) {
          const uint32_t e7 = (v >> 24) & 0x7Fu;
          mx = max(mx, e7);
          orv |= v;
          mn_z = min(mn_z, v ? e7 : 127u);
          posnz |= uint32_t(v - 1u < 0x7FFFFFFFu);
          if (decltype(full)::value || uint32_t(r * 256 + threadIdx.x) < nvalid) {
            mn_a = min(mn_a, e7);
            andv &= v;
          }
        }
      }
    };
    if (nvalid == uint32_t(kZvcTileWords)) tile_stats(std::true_type{});
    else tile_stats(std::false_type{});
    nnz = __reduce_add_sync(0xffffffffu, nnz);
    if (kExp) {
      mn_a = __reduce_min_sync(0xffffffffu, mn_a);
      mx = __reduce_max_sync(0xffffffffu, mx);
      orv = __reduce_or_sync(0xffffffffu, orv) >> 31;
      andv = __reduce_and_sync(0xffffffffu, andv) >> 31;
      mn_z = __reduce_min_sync(0xffffffffu, mn_z);
      posnz = __reduce_or_sync(0xffffffffu, posnz);
    }
    if (lane == 0) {
      red[warp][0] = nnz; red[warp][1] = mn_a; red[warp][2] = mx; red[warp][3] = orv; red[warp][4] = andv;
      red[warp][5] = mn_z; red[warp][6] = posnz;
    }
    __syncthreads();
    // every thread takes the same decision from the 8 warps' partials (no
    // serial thread-0 step, no second barrier)
    uint32_t z = 0, mna = 127, mxa = 0, ora = 0, anda = 1, mnz = 127, posz = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      z += red[k][0];
      if (kExp) {
        mna = min(mna, red[k][1]); mxa = max(mxa, red[k][2]); ora |= red[k][3]; anda &= red[k][4];
        mnz = min(mnz, red[k][5]); posz |= red[k][6];
      }
    }
    const uint32_t mxz = mxa, orz = ora, andz = posz ? 0u : 1u;
    uint32_t mode = kZRaw, bytes = zvc_pad16(4ull * nvalid), n = nvalid, k = 0, sp = 0, sc = 0, em = 0, hoff = 0;
    {
      const uint32_t bm = 512 + zvc_pad16(4ull * z);
      if (bm < bytes) mode = kZMask, bytes = bm, n = z;
      if (kExp) {
        const uint32_t kd = zvc_nbits(mxa - mna), sd = ora != anda;
        const uint32_t ng = (nvalid + 31) / 32;
        const uint32_t bd = 96 * ng + zvc_pad16(4ull * ng * (kd + sd));
        if (bd < bytes) mode = kZExpD, bytes = bd, n = nvalid, k = kd, sp = sd, sc = ora, em = mna, hoff = 96 * ng;
        if (z) {
          const uint32_t km = zvc_nbits(mxz - mnz), sm = orz != andz;
          const uint32_t be = 512 + zvc_pad16(3ull * z) + zvc_pad16((uint64_t(z) * (km + sm) + 7) / 8);
          if (be < bytes) mode = kZExpM, bytes = be, n = z, k = km, sp = sm, sc = orz, em = mnz,
                          hoff = 512 + zvc_pad16(3ull * z);
        }
      }
    }
    const uint32_t info = mode | k << 2 | sp << 6 | sc << 7 | em << 8 | n << 16;
    if (mode == kZExpM) {   // the code plane is OR-ed together: clear it (and the padding) first
      for (uint32_t q = hoff / 4 + threadIdx.x; q < bytes / 4; q += 256) cw[q] = 0u;
      for (uint32_t b = 512u + 3u * n + threadIdx.x; b < hoff; b += 256) chunk[b] = 0;
    } else if (mode == kZExpD) {   // the low plane is written in whole words; the code plane is OR-ed
      for (uint32_t q = hoff / 4 + threadIdx.x; q < bytes / 4; q += 256) cw[q] = 0u;
    }
    const bool masked = mode == kZMask || mode == kZExpM;
    if (masked) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t m = __ballot_sync(0xffffffffu, w16[r] != 0);
        if (lane == 0) cw[r * 8 + warp] = m;
      }
    }
    if (mode != kZRaw) __syncthreads();   // masks complete, planes cleared
    // masked forms: each warp scans the 128 mask popcounts itself; the prefix of
    // mask word r*8 + warp sits in lane 2r + warp/4 at position warp % 4
    uint32_t psel = 0;
    if (masked) {
      const uint32_t c0 = __popc(cw[4 * lane]), c1 = __popc(cw[4 * lane + 1]);
      const uint32_t c2 = __popc(cw[4 * lane + 2]), c3 = __popc(cw[4 * lane + 3]);
      const uint32_t sum = c0 + c1 + c2 + c3;
      uint32_t x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t ex = x - sum;
      const uint32_t pos = warp & 3;
      psel = ex + (pos > 0 ? c0 : 0) + (pos > 1 ? c1 : 0) + (pos > 2 ? c2 : 0);
    }
    if (mode == kZRaw) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t j = r * 256 + threadIdx.x;
        if (j < bytes / 4) cw[j] = w16[r];   // zero past nwords: the padding is deterministic
      }
    } else if (mode == kZMask) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t m = cw[r * 8 + warp];
        const uint32_t base_r = __shfl_sync(0xffffffffu, psel, 2 * r + (warp >> 2));
        if (w16[r] != 0) cw[kZvcMaskWords + base_r + __popc(m & lt)] = w16[r];
      }
      if (threadIdx.x < ((z + 3) & ~3u) - z) cw[kZvcMaskWords + z + threadIdx.x] = 0u;
    } else if (mode == kZExpD) {
      // warp-cooperative: a warp's 32 consecutive words are one group -- their low
      // 24 bits are 96 contiguous bytes (24 aligned words, gathered by shuffles)
      // and their codes are b ballots (bit planes), no shared-memory atomics
      uint32_t* hi = reinterpret_cast<uint32_t*>(chunk + hoff);
      const uint32_t b = k + sp;
      const uint32_t a = (4 * lane) / 3, off = 4 * lane - 3 * a;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t g = r * 8 + warp;
        if (32 * g >= nvalid) break;   // warp-uniform
        const bool valid = g * 32 + lane < nvalid;
        const uint32_t v = w16[r];
        const uint32_t lo = v & 0xFFFFFFu;
        const uint32_t la = __shfl_sync(0xffffffffu, lo, a & 31), lb = __shfl_sync(0xffffffffu, lo, (a + 1) & 31);
        const uint64_t cat = uint64_t(la) | (uint64_t(lb) << 24);
        if (lane < 24) cw[g * 24 + lane] = uint32_t(cat >> (8 * off));
        // codes packed b bits each (the plane was cleared above; two shared-memory
        // ORs at most per word -- measured faster than warp-wide assembly)
        if (valid && b) {
          const uint32_t code = (((v >> 24) & 0x7Fu) - em) | (sp ? (v >> 31) << k : 0u);
          const uint32_t o = (g * 32 + lane) * b, q = o >> 5, sh = o & 31u;
          atomicOr(hi + q, code << sh);
          if (sh + b > 32) atomicOr(hi + q + 1, code >> (32 - sh));
        }
      }
    } else {
      uint32_t* hi = reinterpret_cast<uint32_t*>(chunk + hoff);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t m = cw[r * 8 + warp];
        const uint32_t base_r = __shfl_sync(0xffffffffu, psel, 2 * r + (warp >> 2));
        if (w16[r] != 0) zvc_put_exp(chunk + 512, hi, base_r + __popc(m & lt), w16[r], k, sp, em);
      }
    }
    char* dst = data + t * kZvcSlotBytes;
    if (use_bulk) {
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_s2g(dst, chunk, bytes);
        bulk_commit();
        table[t] = ZvcTile{info, bytes};
      }
    } else {
      __syncthreads();
      const uint4* c4 = reinterpret_cast<const uint4*>(chunk);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (uint32_t q = threadIdx.x; q < bytes / 16; q += 256) st_stream(d4 + q, c4[q]);
      if (threadIdx.x == 0) table[t] = ZvcTile{info, bytes};
    }
  }
  if (use_bulk && threadIdx.x == 0) bulk_wait<0>();
}

// decode: `enc` may live in HBM or in mapped pinned host memory (zero-copy
// swap-in).  Each CTA walks its tiles with a two-deep pipeline: the bulk load
// of tile k+1's chunk is in flight while tile k is expanded from shared memory
// into coalesced HBM stores; tile entries are read one tile further ahead.
__global__ void __launch_bounds__(256) zvc_decode_kernel(const char* __restrict__ enc, uint64_t nwords,
                                                         uint32_t* __restrict__ dst, int use_bulk) {
  extern __shared__ __align__(128) unsigned char zsm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t seg[kZvcMaskWords + 1];
  __shared__ uint32_t s_info[2];
  const uint64_t ntiles = zvc_tiles(nwords);
  const ZvcTile* table = reinterpret_cast<const ZvcTile*>(enc + 64);
  const char* data = enc + zvc_data_pos(ntiles);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  if (use_bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  ZvcTile next{0, 0};   // thread 0: the entry of the tile after the one in flight
  auto issue = [&](uint64_t t, int b, uint32_t bytes) {  // thread 0 only
    mbar_expect_tx(&bar[b], bytes);
    bulk_g2s(zsm + b * kZvcBufBytes, data + t * kZvcSlotBytes, bytes, &bar[b]);
  };
  uint32_t phase0 = 0, phase1 = 0;
  if (threadIdx.x == 0 && blockIdx.x < ntiles) {
    const ZvcTile e0 = table[blockIdx.x];
    s_info[0] = e0.info;
    if (use_bulk) issue(blockIdx.x, 0, e0.bytes);
    if (blockIdx.x + gridDim.x < ntiles) next = table[blockIdx.x + gridDim.x];
  }
  int b = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, b ^= 1) {
    unsigned char* chunk = zsm + b * kZvcBufBytes;
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(chunk);
    __syncthreads();   // s_info of this tile is published; buffer b^1 is free
    const uint32_t info = s_info[b];
    if (use_bulk) {
      const uint64_t tn = t + gridDim.x;
      if (threadIdx.x == 0 && tn < ntiles) {
        s_info[b ^ 1] = next.info;
        issue(tn, b ^ 1, next.bytes);
        if (tn + gridDim.x < ntiles) next = table[tn + gridDim.x];
      }
      if (b == 0) {
        mbar_wait(&bar[0], phase0);
        phase0 ^= 1;
      } else {
        mbar_wait(&bar[1], phase1);
        phase1 ^= 1;
      }
    } else {
      const ZvcTile e = table[t];
      const uint4* s4 = reinterpret_cast<const uint4*>(data + t * kZvcSlotBytes);
      uint4* c4 = reinterpret_cast<uint4*>(chunk);
      for (uint32_t q = threadIdx.x; q < e.bytes / 16; q += 256) c4[q] = ld_stream(s4 + q);
      if (threadIdx.x == 0 && t + gridDim.x < ntiles) s_info[b ^ 1] = table[t + gridDim.x].info;
      __syncthreads();
    }
    const uint32_t mode = info & 3u, k = (info >> 2) & 15u, sp = (info >> 6) & 1u, sc = (info >> 7) & 1u,
                   em = (info >> 8) & 0x7Fu, n = info >> 16;
    const bool masked = mode == kZMask || mode == kZExpM;
    if (masked) {
      if (threadIdx.x < kZvcMaskWords) seg[threadIdx.x] = __popc(cw[threadIdx.x]);
      __syncthreads();
      if (warp == 0) zvc_seg_scan(seg, lane);
      __syncthreads();
    }
    const uint32_t hoff = mode == kZExpD ? 96 * ((n + 31) / 32) : 512 + zvc_pad16(3ull * n);
    const unsigned char* lo = chunk + (mode == kZExpM ? 512 : 0);
    const uint32_t* hi = reinterpret_cast<const uint32_t*>(chunk + hoff);
    const uint64_t base = t * kZvcTileWords;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t j = r * 256 + threadIdx.x;
      const uint64_t i = base + j;
      uint32_t v;
      if (mode == kZRaw) {
        v = cw[j < kZvcTileWords ? j : 0];
      } else if (mode == kZExpD) {
        // word j: low bytes at 3 j (two aligned word loads), code at bit j b (packed)
        const uint32_t sh = (3 * j & 3) * 8, b = k + sp;
        const uint32_t* lw = cw + (3 * j) / 4;
        const uint32_t low = ((lw[0] >> sh) | (sh > 8 ? lw[1] << (32 - sh) : 0u)) & 0xFFFFFFu;
        uint32_t code = 0;
        if (b) {
          const uint32_t o = j * b, q = o >> 5, s2 = o & 31u;
          code = hi[q] >> s2;
          if (s2 + b > 32) code |= hi[q + 1] << (32 - s2);
        }
        const uint32_t e7 = em + (code & ((1u << k) - 1u));
        const uint32_t sg = sp ? (code >> k) & 1u : sc;
        v = i < nwords ? (((sg << 7 | e7) << 24) | low) : 0u;
      } else {
        const uint32_t m = cw[r * 8 + warp];
        const uint32_t p = seg[r * 8 + warp] + __popc(m & lt);
        v = ((m >> lane) & 1u) ? (mode == kZMask ? cw[kZvcMaskWords + p] : zvc_get_exp(lo, hi, p, k, sp, sc, em))
                               : 0u;
      }
      if (i < nwords) dst[i] = v;
    }
  }
}

// -------------------------------------------------------------------------
// Replay payload of one graph op (lms_sim_op, the measured `simulate`): each
// input is checked word by word against the pattern its origin tensor was
// written with (a swap chain must deliver exactly those bytes), each output
// is filled with its own pattern, and the op lasts at least `spin_ns` (the
// node's cost_hint).  Pure HBM streaming: uint4 accesses where aligned.

constexpr int kSimMaxArgs = 8;

struct SimArgs {
  const void* in[kSimMaxArgs];
  void* out[kSimMaxArgs];
  uint64_t in_bytes[kSimMaxArgs], out_bytes[kSimMaxArgs];
  uint32_t in_tag[kSimMaxArgs], out_tag[kSimMaxArgs];
  int n_in, n_out;
};

__device__ __forceinline__ uint32_t sim_word(uint32_t tag, uint64_t i) {
  uint32_t x = tag * 0x9E3779B1u ^ uint32_t(i) * 0x85EBCA77u ^ uint32_t(i >> 32) * 0xC2B2AE3Du;
  x ^= x >> 15;
  return x * 0x2C1B3C6Du;
}

__global__ void __launch_bounds__(256) sim_op_kernel(SimArgs a, uint64_t spin_ns, uint32_t* __restrict__ errors) {
  uint64_t t_start = 0;
  if (spin_ns && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nth = uint64_t(gridDim.x) * blockDim.x;
  uint32_t bad = 0;
  for (int k = 0; k < a.n_in; ++k) {
    const uint32_t* p = static_cast<const uint32_t*>(a.in[k]);
    const uint64_t nw = a.in_bytes[k] / 4;
    const uint32_t tag = a.in_tag[k];
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const uint64_t n4 = nw / 4;
      for (uint64_t i = tid; i < n4; i += nth) {
        const uint4 v = ld_stream(reinterpret_cast<const uint4*>(p) + i);
        bad += (v.x != sim_word(tag, 4 * i)) + (v.y != sim_word(tag, 4 * i + 1)) +
               (v.z != sim_word(tag, 4 * i + 2)) + (v.w != sim_word(tag, 4 * i + 3));
      }
      for (uint64_t i = n4 * 4 + tid; i < nw; i += nth) bad += p[i] != sim_word(tag, i);
    } else {
      for (uint64_t i = tid; i < nw; i += nth) bad += p[i] != sim_word(tag, i);
    }
  }
  for (int k = 0; k < a.n_out; ++k) {
    uint32_t* p = static_cast<uint32_t*>(a.out[k]);
    const uint64_t nw = a.out_bytes[k] / 4;
    const uint32_t tag = a.out_tag[k];
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const uint64_t n4 = nw / 4;
      for (uint64_t i = tid; i < n4; i += nth)
        st_stream(reinterpret_cast<uint4*>(p) + i, make_uint4(sim_word(tag, 4 * i), sim_word(tag, 4 * i + 1),
                                                              sim_word(tag, 4 * i + 2), sim_word(tag, 4 * i + 3)));
      for (uint64_t i = n4 * 4 + tid; i < nw; i += nth) p[i] = sim_word(tag, i);
    } else {
      for (uint64_t i = tid; i < nw; i += nth) p[i] = sim_word(tag, i);
    }
  }
  if (bad) atomicAdd(errors, bad);
  if (spin_ns && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t now = t_start;
    while (now - t_start < spin_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  }
}

}  // namespace lms

// -------------------------------------------------------------------------
// TMA pack/unpack ("rows" layouts): both sides are described by 5-D tensor
// maps with identical logical dims (innermost unit-stride on both); a
// single elected thread per CTA walks boxes through a STAGES-deep ring of
// shared-memory buffers: cp.async.bulk.tensor load (mbarrier completion) ->
// cp.async.bulk.tensor store.  The TMA engine does all address generation,
// so the per-byte instruction cost is ~0 (the SIMT kernels above spend it on
// 64-bit index math).  OOB parts of edge boxes are zero-filled on load and
// clipped on store.  Stage buffers are 1 KiB aligned (TMA needs >= 128 B).

#include <cuda.h>

namespace lms {

struct TmaBoxGrid {
  uint32_t nbox[5];   // boxes per dim (innermost first)
  uint32_t box[5];    // box extent per dim
  uint64_t total;     // product of nbox
};

__device__ __forceinline__ void tma_load_5d(void* smem, const CUtensorMap* map, const int c[5], uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const int c[5], const void* smem) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(smem))
               : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(32) tma_copy_kernel(const __grid_constant__ CUtensorMap src,
                                                      const __grid_constant__ CUtensorMap dst, TmaBoxGrid g,
                                                      uint32_t box_bytes, uint32_t stage_bytes) {
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;  // one thread drives the TMA engine
  for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  fence_mbar_init();
  auto coords = [&](uint64_t b, int c[5]) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t q = uint32_t(b % g.nbox[k]);
      b /= g.nbox[k];
      c[k] = int(q * g.box[k]);
    }
  };
  const uint64_t step = gridDim.x;
  uint64_t next_load = blockIdx.x, next_store = blockIdx.x;
  uint32_t phase_bits = 0;
  int s_load = 0, s_store = 0, inflight = 0;
  int c[5];
  while (inflight < STAGES && next_load < g.total) {
    coords(next_load, c);
    mbar_expect_tx(&bar[s_load], box_bytes);
    tma_load_5d(tsm + size_t(s_load) * stage_bytes, &src, c, &bar[s_load]);
    next_load += step;
    s_load = (s_load + 1) % STAGES;
    ++inflight;
  }
  while (inflight > 0) {
    mbar_wait(&bar[s_store], (phase_bits >> s_store) & 1u);
    phase_bits ^= 1u << s_store;
    coords(next_store, c);
    tma_store_5d(&dst, c, tsm + size_t(s_store) * stage_bytes);
    bulk_commit();
    next_store += step;
    --inflight;
    s_store = (s_store + 1) % STAGES;
    if (next_load < g.total) {
      bulk_wait_read<0>();  // the stage about to be refilled has been read by its store
      coords(next_load, c);
      mbar_expect_tx(&bar[s_load], box_bytes);
      tma_load_5d(tsm + size_t(s_load) * stage_bytes, &src, c, &bar[s_load]);
      next_load += step;
      s_load = (s_load + 1) % STAGES;
      ++inflight;
    }
  }
  bulk_wait<0>();
}

// -------------------------------------------------------------------------
// TMA transpose pack/unpack: the strided side's unit-stride dim is not its
// innermost one (e.g. a channels-last view of an NCHW tensor).  Tiles of
// T x T elements (T * E = 128 B) are loaded by cp.async.bulk.tensor with the
// 128 B swizzle, transposed through shared memory by the CTA (the swizzle
// keeps the row-side accesses conflict-free), and stored by
// cp.async.bulk.tensor with the same swizzle from a second buffer.  One
// elected thread drives the TMA engine; loads run STAGES tiles ahead.

__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t byte_col) {
  return row * 128u + ((((byte_col >> 4) ^ (row & 7u))) << 4) + (byte_col & 15u);
}

// Each warp runs its own two-deep pipeline (no CTA-wide barriers: lane 0
// drives the TMA engine, the warp transposes): the block-synchronous first
// version spent two thirds of its cycles waiting at __syncthreads.
template <int E, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) tma_transpose_kernel(const __grid_constant__ CUtensorMap src,
                                                                   const __grid_constant__ CUtensorMap dst,
                                                                   TmaBoxGrid g) {
  using W = typename Word<E>::T;
  constexpr uint32_t T = 128 / E;
  constexpr uint32_t kTile = T * 128;  // bytes
  extern __shared__ __align__(1024) unsigned char tsm[];
  __shared__ __align__(8) uint64_t bar[WARPS][2];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* in = base + warp * 4 * kTile;   // 2 input tiles, then 2 output tiles
  unsigned char* out = in + 2 * kTile;
  auto coords = [&](uint64_t b, int c[5]) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t q = uint32_t(b % g.nbox[k]);
      b /= g.nbox[k];
      c[k] = int(q * g.box[k]);
    }
  };
  const uint64_t nw = uint64_t(gridDim.x) * WARPS;
  uint64_t t = uint64_t(blockIdx.x) * WARPS + warp;
  int c[5];
  if (lane == 0) {
    mbar_init(&bar[warp][0], 1);
    mbar_init(&bar[warp][1], 1);
    fence_mbar_init();
    if (t < g.total) {
      coords(t, c);
      mbar_expect_tx(&bar[warp][0], kTile);
      tma_load_5d(in, &src, c, &bar[warp][0]);
    }
  }
  __syncwarp();
  uint32_t phases = 0;
  for (uint32_t k = 0; t < g.total; t += nw, ++k) {
    const uint32_t b = k & 1u;
    if (lane == 0 && t + nw < g.total) {  // prefetch the next tile into the other buffer
      coords(t + nw, c);
      mbar_expect_tx(&bar[warp][b ^ 1u], kTile);
      tma_load_5d(in + (b ^ 1u) * kTile, &src, c, &bar[warp][b ^ 1u]);
    }
    mbar_wait(&bar[warp][b], (phases >> b) & 1u);
    phases ^= 1u << b;
    if (lane == 0) bulk_wait_read<1>();  // the store that last read out[b] is done reading
    __syncwarp();
    const unsigned char* A = in + b * kTile;
    unsigned char* B = out + b * kTile;
    // B[r][col] = A[col][r]: lane = col walks a B row (conflict-free stores)
#pragma unroll 8
    for (uint32_t r = 0; r < T; ++r)
      for (uint32_t col = lane; col < T; col += 32)
        *reinterpret_cast<W*>(B + swz128(r, col * E)) = *reinterpret_cast<const W*>(A + swz128(col, r * E));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      coords(t, c);
      int sc[5] = {c[1], c[0], c[2], c[3], c[4]};
      tma_store_5d(&dst, sc, B);
      bulk_commit();
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait<0>();
}

}  // namespace lms
