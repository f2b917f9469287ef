// bsb_common.cuh -- shared device helpers for the B200 ByteStore kernels.
//
// Lane model used by every scan kernel: one warp owns a TILE of 32 blocks
// (1024 rows); lane b owns block b of the tile and keeps that block's 32-bit
// lane masks (gt / eq / result, bit r = row r of the block, LSB first --
// reference bitvector.py:1-6) in registers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bytestore_b200.h"

namespace bsb {

constexpr int kLanes = 32;
constexpr int kTileRows = 1024;
constexpr int kMaxLevels = 8;
constexpr unsigned kFull = 0xffffffffu;

// Status propagation ---------------------------------------------------------
void set_error(const char* where, cudaError_t err);
void set_error_msg(const char* msg);
#define BSB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e__ = (call);                            \
    if (e__ != cudaSuccess) {                            \
      ::bsb::set_error(#call, e__);                      \
      return BSB_ECUDA;                                  \
    }                                                    \
  } while (0)
#define BSB_LAUNCH_CHECK()                               \
  do {                                                   \
    cudaError_t e__ = cudaGetLastError();                \
    if (e__ != cudaSuccess) {                            \
      ::bsb::set_error("kernel launch", e__);            \
      return BSB_ECUDA;                                  \
    }                                                    \
  } while (0)

// First use per process: keep freed stream-ordered allocations in the
// device pool (release threshold = max) so per-call temporaries do not go
// back to the driver at every synchronisation.
void ensure_init();
inline cudaStream_t as_stream(void* s) {
  ensure_init();
  return reinterpret_cast<cudaStream_t>(s);
}

// Grid sizing: persistent grid-stride kernels use (SMs x resident CTAs).
int sm_count();
template <typename K>
int persistent_grid(K kernel, int threads, int64_t work_items_per_cta_iter, int64_t total_items) {
  static thread_local int cached_blocks = -1;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  if (per_sm < 1) per_sm = 1;
  (void)cached_blocks;
  int64_t want = (total_items + work_items_per_cta_iter - 1) / work_items_per_cta_iter;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

// Row swizzle inside one 32-byte block of a byte plane: row r -> byte
// ((r & 7) << 2) | (r >> 3).  Word i (bytes 4i..4i+3) then holds rows
// {i, 8+i, 16+i, 24+i}, which lets cmp_block() build lane masks with
// PRMT + shifted adds and no bit gather.
__host__ __device__ __forceinline__ int swz(int r) { return ((r & 7) << 2) | (r >> 3); }

// 256-bit read-only streaming load (sm_100: LDG.E.NA.ENL2.256.CONSTANT).
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&w)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

// Literal constants for one level of one comparison leg: adding (255 - L)
// to a byte in a 16-bit lane carries into bit 8 iff byte > L; adding
// (256 - L) carries iff byte >= L.
struct LevelLit {
  uint32_t cgt;
  uint32_t cge;
};
__host__ __device__ inline LevelLit make_level_lit(uint32_t byte) {
  LevelLit l;
  l.cgt = (255u - byte) * 0x00010001u;
  l.cge = (256u - byte) * 0x00010001u;
  return l;
}

// Compare the 32 swizzled bytes of one block against one literal byte:
// returns (gt, ge) lane masks in row order.
__device__ __forceinline__ void cmp_block(const uint32_t (&w)[8], LevelLit L, uint32_t& gt,
                                          uint32_t& ge) {
  uint32_t g = 0, e = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);  // [b0, 0, b2, 0]
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);  // [b1, 0, b3, 0]
    const uint32_t gf = __byte_perm(ev + L.cgt, od + L.cgt, 0x7351);  // carry bytes -> 0/1
    const uint32_t ef = __byte_perm(ev + L.cge, od + L.cge, 0x7351);
    g += gf << i;  // byte k, bit i  == row 8k + i
    e += ef << i;
  }
  gt = g;
  ge = e;
}

// cmp_block for PP-VBS levels: a literal byte 0xFF (PPE's right-most pointer
// slot, the first byte of every long code in the skewed columns) has nothing
// above it, so only the >= (here: ==) carries are computed.
__device__ __forceinline__ void cmp_block_vbs(const uint32_t (&w)[8], LevelLit L, uint32_t& gt,
                                              uint32_t& ge) {
  if (L.cgt != 0u) {
    cmp_block(w, L, gt, ge);
    return;
  }
  uint32_t e = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    e += __byte_perm(ev + L.cge, od + L.cge, 0x7351) << i;
  }
  gt = 0u;
  ge = e;
}

// Two literals at once (fused BETWEEN), sharing the byte split.
__device__ __forceinline__ void cmp_block2(const uint32_t (&w)[8], LevelLit A, LevelLit B,
                                           uint32_t& gtA, uint32_t& geA, uint32_t& gtB,
                                           uint32_t& geB) {
  uint32_t ga = 0, ea = 0, gb = 0, eb = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    ga += __byte_perm(ev + A.cgt, od + A.cgt, 0x7351) << i;
    ea += __byte_perm(ev + A.cge, od + A.cge, 0x7351) << i;
    gb += __byte_perm(ev + B.cgt, od + B.cgt, 0x7351) << i;
    eb += __byte_perm(ev + B.cge, od + B.cge, 0x7351) << i;
  }
  gtA = ga;
  geA = ea;
  gtB = gb;
  geB = eb;
}

// Level-1 compares for a lo literal byte 0x00 (the top byte of every small
// rank): everything is >= it, so only the > carries are computed.  Selected
// by a kernel template argument, never by a branch inside the compare.
__device__ __forceinline__ void cmp_block_z(const uint32_t (&w)[8], LevelLit L, uint32_t& gt,
                                            uint32_t& ge) {
  uint32_t g = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    g += __byte_perm(ev + L.cgt, od + L.cgt, 0x7351) << i;
  }
  gt = g;
  ge = kFull;
}
__device__ __forceinline__ void cmp_block2_z(const uint32_t (&w)[8], LevelLit A, LevelLit B,
                                             uint32_t& gtA, uint32_t& geA, uint32_t& gtB,
                                             uint32_t& geB) {
  uint32_t ga = 0, gb = 0, eb = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    ga += __byte_perm(ev + A.cgt, od + A.cgt, 0x7351) << i;
    gb += __byte_perm(ev + B.cgt, od + B.cgt, 0x7351) << i;
    eb += __byte_perm(ev + B.cge, od + B.cge, 0x7351) << i;
  }
  gtA = ga;
  geA = kFull;
  gtB = gb;
  geB = eb;
}

// cmp_block2 for PP-VBS levels: when the hi literal byte is 0xFF only its
// >= carries are needed (nothing is above 0xFF).
__device__ __forceinline__ void cmp_block2_vbs(const uint32_t (&w)[8], LevelLit A, LevelLit B,
                                               uint32_t& gtA, uint32_t& geA, uint32_t& gtB,
                                               uint32_t& geB) {
  if (B.cgt != 0u) {
    cmp_block2(w, A, B, gtA, geA, gtB, geB);
    return;
  }
  uint32_t ga = 0, ea = 0, eb = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    ga += __byte_perm(ev + A.cgt, od + A.cgt, 0x7351) << i;
    ea += __byte_perm(ev + A.cge, od + A.cge, 0x7351) << i;
    eb += __byte_perm(ev + B.cge, od + B.cge, 0x7351) << i;
  }
  gtA = ga;
  geA = ea;
  gtB = 0u;
  geB = eb;
}

// Packed-order compare of 4 consecutive bytes (rank 4i..4i+3): 4-bit masks.
__device__ __forceinline__ uint32_t nib4(uint32_t flags) {
  // flags bytes are 0/1; gather bit 0 of each byte into bits 0..3
  return ((flags * 0x00204081u) >> 21) & 0xFu;
}
__device__ __forceinline__ void cmp_word_packed(uint32_t w, LevelLit L, uint32_t& g4,
                                                uint32_t& e4) {
  const uint32_t ev = __byte_perm(w, 0, 0x4240);
  const uint32_t od = __byte_perm(w, 0, 0x4341);
  // byte order [b0, b1, b2, b3] -> flags bytes in the same order
  g4 = nib4(__byte_perm(ev + L.cgt, od + L.cgt, 0x7351));
  e4 = nib4(__byte_perm(ev + L.cge, od + L.cge, 0x7351));
}

// Hacker's Delight "expand" (pdep) as a 5-stage butterfly.  The stage masks
// depend only on the mask m and are shared by every word expanded with it.
struct ExpandNet {
  uint32_t mv[5];
  uint32_t m0;
};
__device__ __forceinline__ ExpandNet expand_setup(uint32_t m) {
  ExpandNet net;
  net.m0 = m;
  uint32_t mk = ~m << 1;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    uint32_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    const uint32_t mv = mp & m;
    net.mv[i] = mv;
    m = (m ^ mv) | (mv >> (1 << i));
    mk &= ~mp;
  }
  return net;
}
__device__ __forceinline__ uint32_t expand_apply(const ExpandNet& net, uint32_t x) {
#pragma unroll
  for (int i = 4; i >= 0; --i) {
    const uint32_t mv = net.mv[i];
    const uint32_t t = x << (1 << i);
    x = (x & ~mv) | (t & mv);
  }
  return x & net.m0;
}

// Hacker's Delight "compress" (pext) reusing the same stage masks.
__device__ __forceinline__ uint32_t compress_apply(const ExpandNet& net, uint32_t x) {
  x &= net.m0;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const uint32_t t = x & net.mv[i];
    x = (x ^ t) | (t >> (1 << i));
  }
  return x;
}

// Warp-cooperative pext / pdep of ONE 32-bit word pair (m, x identical in
// every lane; lane = bit position): a handful of instructions per word, used
// for the few blocks of a tile whose masks are not trivial.
__device__ __forceinline__ uint32_t warp_pext(uint32_t m, uint32_t x, int lane) {
  const uint32_t bit = 1u << lane;
  const uint32_t v = ((m & x & bit) != 0) ? (1u << __popc(m & (bit - 1u))) : 0u;
  return __reduce_or_sync(kFull, v);
}
__device__ __forceinline__ uint32_t warp_pdep(uint32_t m, uint32_t x, int lane) {
  const uint32_t bit = 1u << lane;
  return __ballot_sync(kFull, (m & bit) && ((x >> __popc(m & (bit - 1u))) & 1u));
}

// Warp-inclusive prefix sum (lane order).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// Finalize an operator from (gt, eq, valid) -- reference vbs.py:179-197.
__device__ __forceinline__ uint32_t finalize_op(int op, uint32_t gt, uint32_t eq,
                                                uint32_t valid) {
  switch (op) {
    case BSB_GT: return gt;
    case BSB_GE: return gt | eq;
    case BSB_EQ: return eq;
    case BSB_NE: return valid & ~eq;
    case BSB_LT: return valid & ~(gt | eq);
    default: return valid & ~gt;  // BSB_LE
  }
}

// Device error word bits of the row-id lookups (err_dev).
constexpr unsigned int kErrNotFound = 1u;  // padded code not in the dictionary -> LookupError
constexpr unsigned int kErrIndex = 2u;     // row id outside [0, n_rows)        -> IndexError

__device__ __forceinline__ uint32_t tail_valid(int64_t block, int64_t n_rows) {
  const int64_t r0 = block * 32;
  if (r0 + 32 <= n_rows) return kFull;
  if (r0 >= n_rows) return 0u;
  return (1u << (unsigned)(n_rows - r0)) - 1u;
}

}  // namespace bsb
