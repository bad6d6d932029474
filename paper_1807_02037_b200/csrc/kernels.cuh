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

template <bool PACK, int E>
__global__ void __launch_bounds__(256) transpose_kernel(char* __restrict__ dst, const char* __restrict__ src,
                                                        Strided d, int cd, int64_t batches) {
  using T = typename Word<E>::T;
  __shared__ T tile[32][33];
  const int last = d.ndim - 1;
  const int64_t nA = d.sizes[cd], nB = d.sizes[last];
  const int64_t tilesA = (nA + 31) / 32, tilesB = (nB + 31) / 32;
  const int64_t ntiles = batches * tilesA * tilesB;
  // logical (row-major) strides of the contiguous side
  int64_t cstride[kMaxDims];
  {
    int64_t acc = 1;
    for (int k = kMaxDims - 1; k >= 0; --k) {
      if (k < d.ndim) { cstride[k] = acc; acc *= d.sizes[k]; }
    }
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t b = t / (tilesA * tilesB);
    int64_t rem = t - b * tilesA * tilesB;
    int64_t a0 = (rem / tilesB) * 32, b0 = (rem % tilesB) * 32;
    // batch index -> offsets over the dims other than cd and last
    int64_t soff = 0, coff = 0, bi = b;
    for (int k = last - 1; k >= 0; --k) {
      if (k == cd) continue;
      int64_t s = d.sizes[k];
      int64_t q = bi / s, x = bi - q * s;
      soff += x * d.strides[k];
      coff += x * cstride[k];
      bi = q;
    }
    const T* sw = reinterpret_cast<const T*>(src);
    T* dw = reinterpret_cast<T*>(dst);
    // phase 1 reads coalesced on the source side, phase 2 writes coalesced on
    // the destination side; the strided side is unit-stride along cd, the
    // contiguous side along the last dim.
    if (PACK) {
      for (int j = ty; j < 32; j += 8) {
        int64_t ia = a0 + tx, ib = b0 + j;
        if (ia < nA && ib < nB) tile[j][tx] = sw[soff + ia * d.strides[cd] + ib * d.strides[last]];
      }
      __syncthreads();
      for (int j = ty; j < 32; j += 8) {
        int64_t ia = a0 + j, ib = b0 + tx;
        if (ia < nA && ib < nB) dw[coff + ia * cstride[cd] + ib] = tile[tx][j];
      }
    } else {
      for (int j = ty; j < 32; j += 8) {
        int64_t ia = a0 + j, ib = b0 + tx;
        if (ia < nA && ib < nB) tile[j][tx] = sw[coff + ia * cstride[cd] + ib];
      }
      __syncthreads();
      for (int j = ty; j < 32; j += 8) {
        int64_t ia = a0 + tx, ib = b0 + j;
        if (ia < nA && ib < nB) dw[soff + ia * d.strides[cd] + ib * d.strides[last]] = tile[tx][j];
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
// ZVC: lossless zero-value compression over 32-bit words.
//
// Stream layout (all offsets in bytes from the start, 16B aligned):
//   [0, 64)                 header  {magic, mode, nwords, ntiles, total_nnz, ...}
//   [64, 64+4*T16)          per-tile value offsets (words), T16 = ntiles rounded to 4
//   [.., +512*ntiles)       per-tile bitmask, 128 words per tile
//   [.., +4*total_nnz)      packed nonzero words, tile order
// A tile is 4096 words (16 KiB).  mode 1 = ZVC, mode 0 = raw fallback (the
// words follow the header directly) chosen on device when compression would
// not shrink the stream.

constexpr int kZvcTileWords = 4096;
constexpr int kZvcMaskWords = kZvcTileWords / 32;  // 128
constexpr uint32_t kZvcMagic = 0x5A564331u;          // "ZVC1"

struct ZvcHeader {
  uint32_t magic, mode;
  uint64_t nwords, ntiles, total_nnz, bytes;
  uint64_t pad[3];
};
static_assert(sizeof(ZvcHeader) == 64, "header is 64 bytes");

__host__ __device__ inline uint64_t zvc_tiles(uint64_t nwords) {
  return (nwords + kZvcTileWords - 1) / kZvcTileWords;
}
__host__ __device__ inline uint64_t zvc_off_bytes(uint64_t ntiles) { return ((ntiles + 3) / 4) * 16; }
__host__ __device__ inline uint64_t zvc_mask_pos(uint64_t ntiles) { return 64 + zvc_off_bytes(ntiles); }
__host__ __device__ inline uint64_t zvc_vals_pos(uint64_t ntiles) {
  return zvc_mask_pos(ntiles) + ntiles * kZvcMaskWords * 4;
}
__host__ __device__ inline uint64_t zvc_bound(uint64_t nwords) {
  uint64_t t = zvc_tiles(nwords);
  uint64_t a = zvc_vals_pos(t) + nwords * 4;
  uint64_t b = 64 + nwords * 4;
  a = a > b ? a : b;
  return (a + 15) / 16 * 16;
}

// pass 1: nonzero count per tile
__global__ void __launch_bounds__(256) zvc_count_kernel(const uint32_t* __restrict__ src, uint64_t nwords,
                                                        uint32_t* __restrict__ counts) {
  __shared__ uint32_t red[8];
  const uint64_t ntiles = zvc_tiles(nwords);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * kZvcTileWords;
    uint32_t c = 0;
    if (base + kZvcTileWords <= nwords) {
      const uint4* s4 = reinterpret_cast<const uint4*>(src + base);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint4 v = ld_stream(s4 + threadIdx.x + k * 256);
        c += (v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0);
      }
    } else {
      for (uint64_t i = base + threadIdx.x; i < nwords; i += 256) c += src[i] != 0;
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

// pass 2 (one CTA): exclusive scan of tile counts -> offsets, write header.
// `offsets` is device scratch; the header and offsets also go to `out`.
__global__ void __launch_bounds__(1024) zvc_scan_kernel(const uint32_t* __restrict__ counts, uint64_t nwords,
                                                        uint32_t* __restrict__ offsets, char* __restrict__ out) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  const uint64_t ntiles = zvc_tiles(nwords);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += 1024) {
    uint64_t i = base + threadIdx.x;
    uint32_t v = i < ntiles ? counts[i] : 0;
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
    uint32_t warp_base = (threadIdx.x >> 5) ? warp_tot[(threadIdx.x >> 5) - 1] : 0;
    uint32_t excl = carry + warp_base + x - v;
    if (i < ntiles) offsets[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint64_t total = carry;
    ZvcHeader h{};
    h.magic = kZvcMagic;
    h.nwords = nwords;
    h.ntiles = ntiles;
    h.total_nnz = total;
    uint64_t zbytes = zvc_vals_pos(ntiles) + total * 4;
    uint64_t rbytes = 64 + nwords * 4;
    h.mode = zbytes < rbytes ? 1u : 0u;
    h.bytes = h.mode ? zbytes : rbytes;
    // the encode kernel reads the mode from the scratch copy
    offsets[ntiles] = h.mode;
    const uint4* hs = reinterpret_cast<const uint4*>(&h);
    uint4* ho = reinterpret_cast<uint4*>(out);
    for (int k = 0; k < 4; ++k) ho[k] = hs[k];
  }
  __syncthreads();
  // offsets table to the output (only meaningful in mode 1)
  uint32_t* oo = reinterpret_cast<uint32_t*>(out + 64);
  for (uint64_t i = threadIdx.x; i < ntiles; i += 1024) oo[i] = offsets[i];
}

// pass 3: per tile, compact the nonzero words through shared memory and
// write bitmask + values with 16B stores (or the raw words in mode 0).
__global__ void __launch_bounds__(256) zvc_encode_kernel(const uint32_t* __restrict__ src, uint64_t nwords,
                                                         const uint32_t* __restrict__ offsets,
                                                         char* __restrict__ out) {
  __shared__ uint32_t vals[kZvcTileWords];
  __shared__ uint32_t mask[kZvcMaskWords];
  __shared__ uint32_t seg[kZvcMaskWords + 1];
  const uint64_t ntiles = zvc_tiles(nwords);
  const uint32_t mode = offsets[ntiles];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (mode == 0) {
    // raw fallback: words after the header, 16B body + word tail
    uint4* o4 = reinterpret_cast<uint4*>(out + 64);
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint64_t n16 = nwords / 4;
    for (uint64_t i = uint64_t(blockIdx.x) * 256 + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * 256)
      st_stream(o4 + i, ld_stream(s4 + i));
    if (blockIdx.x == 0) {
      uint32_t* ow = reinterpret_cast<uint32_t*>(out + 64);
      for (uint64_t i = n16 * 4 + threadIdx.x; i < nwords; i += 256) ow[i] = src[i];
    }
    return;
  }
  uint32_t* mask_out = reinterpret_cast<uint32_t*>(out + zvc_mask_pos(ntiles));
  uint32_t* vals_out = reinterpret_cast<uint32_t*>(out + zvc_vals_pos(ntiles));
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * kZvcTileWords;
    // round r covers words [r*256, r*256+256); warp w of round r is segment r*8+w
    uint32_t w16[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      uint64_t i = base + r * 256 + threadIdx.x;
      w16[r] = i < nwords ? __ldg(src + i) : 0u;
      uint32_t m = __ballot_sync(0xffffffffu, w16[r] != 0);
      if (lane == 0) { mask[r * 8 + warp] = m; seg[r * 8 + warp] = __popc(m); }
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan over the 128 segment counts
      uint32_t a = seg[lane * 4], b = seg[lane * 4 + 1], c = seg[lane * 4 + 2], e = seg[lane * 4 + 3];
      uint32_t s = a + b + c + e, x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      uint32_t ex = x - s;
      seg[lane * 4] = ex; seg[lane * 4 + 1] = ex + a; seg[lane * 4 + 2] = ex + a + b;
      seg[lane * 4 + 3] = ex + a + b + c;
      if (lane == 31) seg[kZvcMaskWords] = x;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      uint32_t m = mask[r * 8 + warp];
      if (w16[r] != 0) vals[seg[r * 8 + warp] + __popc(m & ((1u << lane) - 1u))] = w16[r];
    }
    __syncthreads();
    // bitmask: 128 words = 32 x 16B
    if (threadIdx.x < 32)
      st_stream(reinterpret_cast<uint4*>(mask_out + t * kZvcMaskWords) + threadIdx.x,
                reinterpret_cast<const uint4*>(mask)[threadIdx.x]);
    // values: head words until 16B aligned, 16B body, tail words
    const uint32_t n = seg[kZvcMaskWords];
    const uint64_t o = offsets[t];
    uint32_t* dstw = vals_out + o;
    uint32_t head = (uint32_t)((4 - (o & 3)) & 3);
    if (head > n) head = n;
    if (threadIdx.x < head) dstw[threadIdx.x] = vals[threadIdx.x];
    const uint32_t body16 = (n - head) / 4;
    // shared-memory source is only 4B aligned after `head` words: assemble in registers
    for (uint32_t k = threadIdx.x; k < body16; k += 256) {
      const uint32_t* sv = vals + head + 4 * k;
      st_stream(reinterpret_cast<uint4*>(dstw + head) + k, make_uint4(sv[0], sv[1], sv[2], sv[3]));
    }
    for (uint32_t k = head + body16 * 4 + threadIdx.x; k < n; k += 256) dstw[k] = vals[k];
    __syncthreads();
  }
}

// decode: `enc` is the whole stream already in HBM (H2D-staged).
__global__ void __launch_bounds__(256) zvc_decode_kernel(const char* __restrict__ enc, uint64_t nwords,
                                                         uint32_t* __restrict__ dst) {
  __shared__ uint32_t mask[kZvcMaskWords];
  __shared__ uint32_t seg[kZvcMaskWords];
  const ZvcHeader* h = reinterpret_cast<const ZvcHeader*>(enc);
  const uint64_t ntiles = zvc_tiles(nwords);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (h->mode == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(enc + 64);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    uint64_t n16 = nwords / 4;
    for (uint64_t i = uint64_t(blockIdx.x) * 256 + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * 256)
      d4[i] = ld_stream(s4 + i);
    if (blockIdx.x == 0) {
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(enc + 64);
      for (uint64_t i = n16 * 4 + threadIdx.x; i < nwords; i += 256) dst[i] = sw[i];
    }
    return;
  }
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(enc + 64);
  const uint32_t* mask_in = reinterpret_cast<const uint32_t*>(enc + zvc_mask_pos(ntiles));
  const uint32_t* vals_in = reinterpret_cast<const uint32_t*>(enc + zvc_vals_pos(ntiles));
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x < kZvcMaskWords) {
      uint32_t m = mask_in[t * kZvcMaskWords + threadIdx.x];
      mask[threadIdx.x] = m;
      seg[threadIdx.x] = __popc(m);
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t a = seg[lane * 4], b = seg[lane * 4 + 1], c = seg[lane * 4 + 2], e = seg[lane * 4 + 3];
      uint32_t s = a + b + c + e, x = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      uint32_t ex = x - s;
      seg[lane * 4] = ex; seg[lane * 4 + 1] = ex + a; seg[lane * 4 + 2] = ex + a + b;
      seg[lane * 4 + 3] = ex + a + b + c;
    }
    __syncthreads();
    const uint32_t* tv = vals_in + offs[t];
    const uint64_t base = t * kZvcTileWords;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      uint64_t i = base + r * 256 + threadIdx.x;
      uint32_t m = mask[r * 8 + warp];
      uint32_t v = ((m >> lane) & 1u) ? tv[seg[r * 8 + warp] + __popc(m & ((1u << lane) - 1u))] : 0u;
      if (i < nwords) dst[i] = v;
    }
    __syncthreads();
  }
}

}  // namespace lms
