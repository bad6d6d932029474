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
//   zvc_*         lossless zero-value compression of 32-bit words:
//                 count -> scan -> encode straight into pinned memory, and
//                 decode from an H2D-staged stream back into HBM
#pragma once

#include <cstdint>
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
// ZVC: lossless zero-value compression over 32-bit words (stream format v2).
//
// A swapped activation is compressed on its way out (SM kernels writing
// straight into mapped pinned memory) and decompressed on its way in (SM
// kernels reading straight out of pinned memory), so only the compressed
// bytes cross the host link and no device staging buffer is needed.
//
// Stream layout (bytes from the start; every region 16 B aligned):
//   [0, 64)                  header {magic "ZVC2", mode, nwords, ntiles, total_nnz, bytes, data_pos}
//   [64, data_pos)           u32 chunk offsets, ntiles+1 entries, in 16 B units from data_pos
//   [data_pos, bytes)        one chunk per tile, in tile order:
//                              128-word bitmask (bit j of word s: word 32s+j of the tile is nonzero)
//                              the tile's nonzero words in order, zero-padded to 16 B
// A tile is 4096 words (16 KiB).  mode 0 = raw: the words follow the header
// directly; the scan kernel picks it on the device when compression would
// not shrink the stream.  Words past nwords in the last tile encode as zero.

constexpr int kZvcTileWords = 4096;
constexpr int kZvcMaskWords = kZvcTileWords / 32;                  // 128
constexpr int kZvcChunkWords = kZvcMaskWords + kZvcTileWords;       // worst-case chunk (4224 words)
constexpr int kZvcSmemBytes = 2 * kZvcChunkWords * 4;               // double-buffered chunks
constexpr uint32_t kZvcMagic = 0x3243565Au;                          // "ZVC2"

struct ZvcHeader {
  uint32_t magic, mode;
  uint64_t nwords, ntiles, total_nnz, bytes, data_pos;
  uint64_t pad[2];
};
static_assert(sizeof(ZvcHeader) == 64, "header is 64 bytes");

__host__ __device__ inline uint64_t zvc_tiles(uint64_t nwords) {
  return (nwords + kZvcTileWords - 1) / kZvcTileWords;
}
__host__ __device__ inline uint64_t zvc_data_pos(uint64_t ntiles) { return 64 + ((ntiles + 1 + 3) / 4) * 16; }
__host__ __device__ inline uint64_t zvc_raw_bytes(uint64_t nwords) { return 64 + (nwords * 4 + 15) / 16 * 16; }
__host__ __device__ inline uint64_t zvc_bound(uint64_t nwords) {
  const uint64_t t = zvc_tiles(nwords);
  const uint64_t a = zvc_data_pos(t) + t * uint64_t(kZvcChunkWords) * 4;  // every tile dense
  const uint64_t b = zvc_raw_bytes(nwords);
  return a > b ? a : b;
}

// pass 1: nonzero words per tile (HBM read; the source stays on the device)
__global__ void __launch_bounds__(256) zvc_count_kernel(const uint32_t* __restrict__ src, uint64_t nwords,
                                                        uint32_t* __restrict__ counts) {
  __shared__ uint32_t red[8];
  const uint64_t ntiles = zvc_tiles(nwords);
  const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * kZvcTileWords;
    uint32_t c = 0;
    if (vec && base + kZvcTileWords <= nwords) {
      const uint4* s4 = reinterpret_cast<const uint4*>(src + base);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint4 v = ld_stream(s4 + threadIdx.x + k * 256);
        c += (v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0);
      }
    } else {
      const uint64_t end = base + kZvcTileWords < nwords ? base + kZvcTileWords : nwords;
      for (uint64_t i = base + threadIdx.x; i < end; i += 256) c += src[i] != 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int w = 0; w < 8; ++w) s += red[w];
      counts[t] = s;
    }
    __syncthreads();
  }
}

// pass 2 (one CTA): chunk sizes -> exclusive offsets; header and offset table
// go to `out`; offsets[ntiles+1] carries the mode to the encode kernel.
__global__ void __launch_bounds__(1024) zvc_scan_kernel(const uint32_t* __restrict__ counts, uint64_t nwords,
                                                        uint32_t* __restrict__ offsets, char* __restrict__ out) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  __shared__ unsigned long long nnz_tot;
  const uint64_t ntiles = zvc_tiles(nwords);
  if (threadIdx.x == 0) {
    carry = 0;
    nnz_tot = 0;
  }
  __syncthreads();
  uint64_t my_nnz = 0;
  for (uint64_t base = 0; base < ntiles; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t nnz = i < ntiles ? counts[i] : 0;
    my_nnz += nnz;
    const uint32_t v = i < ntiles ? kZvcMaskWords / 4 + (nnz + 3) / 4 : 0;  // chunk size, 16 B units
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = warp_tot[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      warp_tot[threadIdx.x] = w;  // inclusive
    }
    __syncthreads();
    const uint32_t warp_base = (threadIdx.x >> 5) ? warp_tot[(threadIdx.x >> 5) - 1] : 0;
    const uint32_t excl = carry + warp_base + x - v;
    if (i < ntiles) offsets[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  atomicAdd(&nnz_tot, (unsigned long long)my_nnz);
  __syncthreads();
  uint32_t* table = reinterpret_cast<uint32_t*>(out + 64);
  if (threadIdx.x == 0) {
    ZvcHeader h{};
    h.magic = kZvcMagic;
    h.nwords = nwords;
    h.ntiles = ntiles;
    h.total_nnz = nnz_tot;
    h.data_pos = zvc_data_pos(ntiles);
    const uint64_t zbytes = h.data_pos + uint64_t(carry) * 16;
    const uint64_t rbytes = zvc_raw_bytes(nwords);
    h.mode = zbytes < rbytes ? 1u : 0u;
    h.bytes = h.mode ? zbytes : rbytes;
    offsets[ntiles] = carry;
    offsets[ntiles + 1] = h.mode;
    const uint4* hs = reinterpret_cast<const uint4*>(&h);
    uint4* ho = reinterpret_cast<uint4*>(out);
    for (int k = 0; k < 4; ++k) ho[k] = hs[k];
    if (h.mode) table[ntiles] = carry;
  }
  __syncthreads();
  if (offsets[ntiles + 1])
    for (uint64_t i = threadIdx.x; i < ntiles; i += 1024) table[i] = offsets[i];
}

// raw mode body: 16 B words after the header (grid-stride), word tail by CTA 0
__device__ __forceinline__ void zvc_raw_copy(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                                             uint64_t nwords) {
  const uint64_t n16 = nwords / 4;
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  const uint64_t nth = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * nth < n16; i += 4 * nth) {
    uint4 a = ld_stream(s4 + i), b = ld_stream(s4 + i + nth);
    uint4 c = ld_stream(s4 + i + 2 * nth), e = ld_stream(s4 + i + 3 * nth);
    st_stream(d4 + i, a); st_stream(d4 + i + nth, b);
    st_stream(d4 + i + 2 * nth, c); st_stream(d4 + i + 3 * nth, e);
  }
  for (; i < n16; i += nth) st_stream(d4 + i, ld_stream(s4 + i));
  if (blockIdx.x == 0)
    for (uint64_t k = n16 * 4 + threadIdx.x; k < nwords; k += blockDim.x) dst[k] = src[k];
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

// pass 3: per tile, bitmask + compacted nonzeros assembled in shared memory,
// then one bulk store of the whole chunk (TMA when use_bulk, else 16 B STG).
// Double-buffered: tile k+1 is compacted while tile k's chunk is in flight.
__global__ void __launch_bounds__(256) zvc_encode_kernel(const uint32_t* __restrict__ src, uint64_t nwords,
                                                         const uint32_t* __restrict__ offsets,
                                                         char* __restrict__ out, int use_bulk) {
  extern __shared__ __align__(128) uint32_t zsm[];
  __shared__ uint32_t seg[kZvcMaskWords + 1];
  const uint64_t ntiles = zvc_tiles(nwords);
  if (offsets[ntiles + 1] == 0) {  // raw mode
    zvc_raw_copy(reinterpret_cast<uint32_t*>(out + 64), src, nwords);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  char* data = out + zvc_data_pos(ntiles);
  int buf = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
    uint32_t* chunk = zsm + buf * kZvcChunkWords;
    if (use_bulk && threadIdx.x == 0) bulk_wait_read<1>();  // the store that last read this buffer
    __syncthreads();
    const uint64_t base = t * kZvcTileWords;
    uint32_t w16[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t i = base + r * 256 + threadIdx.x;
      w16[r] = i < nwords ? __ldg(src + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t m = __ballot_sync(0xffffffffu, w16[r] != 0);
      if (lane == 0) {
        chunk[r * 8 + warp] = m;
        seg[r * 8 + warp] = __popc(m);
      }
    }
    __syncthreads();
    if (warp == 0) zvc_seg_scan(seg, lane);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t m = chunk[r * 8 + warp];
      if (w16[r] != 0) chunk[kZvcMaskWords + seg[r * 8 + warp] + __popc(m & ((1u << lane) - 1u))] = w16[r];
    }
    const uint32_t n = seg[kZvcMaskWords];
    const uint32_t padded = (n + 3) & ~3u;
    if (threadIdx.x < padded - n) chunk[kZvcMaskWords + n + threadIdx.x] = 0u;
    const uint32_t bytes = (kZvcMaskWords + padded) * 4;
    char* dst = data + uint64_t(offsets[t]) * 16;
    if (use_bulk) {
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_s2g(dst, chunk, bytes);
        bulk_commit();
      }
    } else {
      __syncthreads();
      const uint4* c4 = reinterpret_cast<const uint4*>(chunk);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      for (uint32_t k = threadIdx.x; k < bytes / 16; k += 256) st_stream(d4 + k, c4[k]);
    }
  }
  if (use_bulk && threadIdx.x == 0) bulk_wait<0>();
}

// decode: `enc` may live in HBM or in mapped pinned host memory (zero-copy
// swap-in).  Each CTA walks its tiles with a two-deep pipeline: the bulk
// load of tile k+1's chunk is in flight while tile k is expanded from shared
// memory into coalesced HBM stores.
__global__ void __launch_bounds__(256) zvc_decode_kernel(const char* __restrict__ enc, uint64_t nwords,
                                                         uint32_t* __restrict__ dst, int use_bulk) {
  extern __shared__ __align__(128) uint32_t zsm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t seg[kZvcMaskWords + 1];
  __shared__ uint32_t s_mode;
  const ZvcHeader* h = reinterpret_cast<const ZvcHeader*>(enc);
  if (threadIdx.x == 0) s_mode = h->mode;
  __syncthreads();
  if (s_mode == 0) {
    zvc_raw_copy(dst, reinterpret_cast<const uint32_t*>(enc + 64), nwords);
    return;
  }
  const uint64_t ntiles = zvc_tiles(nwords);
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(enc + 64);
  const char* data = enc + zvc_data_pos(ntiles);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (use_bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  auto issue = [&](uint64_t t, int b) {  // thread 0 only
    const uint32_t a = offs[t], e = offs[t + 1];
    const uint32_t bytes = (e - a) * 16;
    mbar_expect_tx(&bar[b], bytes);
    bulk_g2s(zsm + b * kZvcChunkWords, data + uint64_t(a) * 16, bytes, &bar[b]);
  };
  uint32_t phase0 = 0, phase1 = 0;
  if (use_bulk && threadIdx.x == 0 && blockIdx.x < ntiles) issue(blockIdx.x, 0);
  int b = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, b ^= 1) {
    uint32_t* chunk = zsm + b * kZvcChunkWords;
    if (use_bulk) {
      const uint64_t tn = t + gridDim.x;
      if (threadIdx.x == 0 && tn < ntiles) issue(tn, b ^ 1);
      if (b == 0) {
        mbar_wait(&bar[0], phase0);
        phase0 ^= 1;
      } else {
        mbar_wait(&bar[1], phase1);
        phase1 ^= 1;
      }
    } else {
      const uint32_t a = offs[t], e = offs[t + 1];
      const uint4* s4 = reinterpret_cast<const uint4*>(data + uint64_t(a) * 16);
      uint4* c4 = reinterpret_cast<uint4*>(chunk);
      for (uint32_t k = threadIdx.x; k < e - a; k += 256) c4[k] = ld_stream(s4 + k);
      __syncthreads();
    }
    if (threadIdx.x < kZvcMaskWords) seg[threadIdx.x] = __popc(chunk[threadIdx.x]);
    __syncthreads();
    if (warp == 0) zvc_seg_scan(seg, lane);
    __syncthreads();
    const uint64_t base = t * kZvcTileWords;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t i = base + r * 256 + threadIdx.x;
      const uint32_t m = chunk[r * 8 + warp];
      const uint32_t v =
          ((m >> lane) & 1u) ? chunk[kZvcMaskWords + seg[r * 8 + warp] + __popc(m & ((1u << lane) - 1u))] : 0u;
      if (i < nwords) dst[i] = v;
    }
    __syncthreads();  // chunk buffer b is free for the load issued two tiles from now
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
