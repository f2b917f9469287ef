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

// Grid sizing: persistent grid-stride kernels use (SMs x resident CTAs),
// optionally capped at ctas_per_sm_cap() CTAs per SM (bsb_tune
// "ctas_per_sm": leaves room on every SM for a kernel of another stream --
// e.g. an ALU-bound PP-VBS scan next to a DRAM-bound ByteSlice scan).
int sm_count();
int ctas_per_sm_cap();  // 0 = no cap
template <typename K>
int persistent_grid(K kernel, int threads, int64_t work_items_per_cta_iter, int64_t total_items) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  if (per_sm < 1) per_sm = 1;
  const int capc = ctas_per_sm_cap();
  if (capc > 0 && per_sm > capc) per_sm = capc;
  int64_t want = (total_items + work_items_per_cta_iter - 1) / work_items_per_cta_iter;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

// 256-bit read-only streaming load (sm_100: LDG.E.NA.ENL2.256.CONSTANT).
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&w)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

// 256-bit load of a sparse, dependent sector (a level read only for blocks
// with tied rows): the L2::64B hint keeps the L2 from fetching a whole 128-B
// line from DRAM for one 32-B sector.
__device__ __forceinline__ void ldg256_sparse(const void* p, uint32_t (&w)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

// Same load without "volatile": the compiler may hoist it above independent
// work (row gathers issue every level's sector before using any of them).
__device__ __forceinline__ void ldg256_free(const void* p, uint32_t (&w)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

// bsb_gather.cu: the sampled order check (*unsorted_dev = 1 when a sampled
// adjacent pair descends, else 0) and the bucket partition into row |
// position << 32 pairs, every kernel gated on *gate != 0 (gate NULL: always).
int rows_order_check(const int64_t* rows, int64_t n_ids, uint32_t* unsorted_dev, cudaStream_t s);
void rows_order_check_launch(const int64_t* rows, int64_t n_ids, uint32_t* unsorted_dev,
                             cudaStream_t s);  // the kernel alone (word already zero)
int rows_bucket_gated(const int64_t* rows, int64_t n_ids, int64_t n_rows, uint64_t* pairs,
                      const uint32_t* gate, cudaStream_t s);
// The same check with the verdict read by the HOST from a mapped word (a poll
// of a few microseconds, no stream synchronisation): 0 = looks ascending, 1 =
// not, -1 = not taken (the stream is capturing or has work queued, or the
// poll timed out) -- the caller then leaves the choice to the device.
int rows_order_poll(const int64_t* rows, int64_t n_ids, cudaStream_t s);

// Device-side gate of a kernel that is one of two alternatives chosen by a
// device word (no host synchronisation, graph-capturable): the kernel runs
// when gate is NULL or (*gate != 0) == want.
__device__ __forceinline__ bool gate_closed(const uint32_t* gate, bool want) {
  return gate && (__ldg(gate) != 0) != want;
}

// 1-D TMA bulk copies global -> shared memory, completion on an mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Bit-plane block layout of a byte plane ("BP32").  Every byte plane of the
// device layouts (ByteSlice slices, the PP-VBS first slice, the SLICED deep
// planes) stores the 32 bytes of one 32-row block -- exactly one 32-byte DRAM
// sector, as in the reference's byte slices -- as 8 uint32 words:
//   word k (k = 0..7) = bit (7 - k) of the byte of every row, bit r = row r.
// The bytes, the sectors a scan touches and the early-stopping decisions are
// the reference's (byteslice.py:56-106, vbs.py:222-289); only the order of the
// bits inside a sector differs.  One 256-bit load gives a lane its block's 8
// words, and a comparison with a literal byte is a carry chain over the bit
// planes: x >= T  <=>  x + (256 - T) carries out of 8 bits, and with the
// addend bits a_p as all-zero / all-one masks each carry step is one
// majority LOP3 for 32 rows at once:  c_{p+1} = maj(x_p, a_p, c_p).
// Results come out as row-ordered lane masks: no byte split, no gather.
// (Round 1 stored the bytes row-swizzled and compared them with SWAR carry
// tricks: ~10 integer instructions per 4 bytes per threshold; the carry
// chain is 8 per 32 bytes.)

// Addend masks of one threshold: m[p] = bit p of the addend ? ~0 : 0.
struct PlaneLit {
  uint32_t m[8];
};
// Addend for "x > L" / "x >= L" of a literal byte L: a = 255 - L, carry-in
// 0 (>) or 1 (>=).
__host__ inline PlaneLit make_plane_lit(uint32_t byte) {
  PlaneLit l;
  const uint32_t a = 255u - (byte & 0xFFu);
  for (int p = 0; p < 8; ++p) l.m[p] = ((a >> p) & 1u) ? kFull : 0u;
  return l;
}
// Threshold "x >= t" for t in 0..256: addend (256 - t) & 255 with carry-in
// 1 only for t == 0 (everything).
struct PlaneThr {
  PlaneLit a;
  uint32_t c0;
};
__host__ inline PlaneThr make_plane_thr(int t) {
  PlaneThr r;
  const uint32_t add = t == 0 ? 255u : (uint32_t)(256 - t) & 0xFFu;
  for (int p = 0; p < 8; ++p) r.a.m[p] = ((add >> p) & 1u) ? kFull : 0u;
  r.c0 = t == 0 ? kFull : 0u;
  return r;
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (c & (a | b));  // one LOP3 (0xE8)
}

// Carry out of x + a + c0 over the 8 bit planes (LSB plane = word 7).
__device__ __forceinline__ uint32_t bp_carry(const uint32_t (&w)[8], const PlaneLit& L,
                                             uint32_t c0) {
  uint32_t c = c0;
#pragma unroll
  for (int p = 0; p < 8; ++p) c = maj3(w[7 - p], L.m[p], c);
  return c;
}

// One literal byte: gt = [x > L], ge = [x >= L], row-ordered lane masks.
__device__ __forceinline__ void cmp_block(const uint32_t (&w)[8], const PlaneLit& L,
                                          uint32_t& gt, uint32_t& ge) {
  gt = bp_carry(w, L, 0u);
  ge = bp_carry(w, L, kFull);
}
// Two literals at once (fused BETWEEN).
__device__ __forceinline__ void cmp_block2(const uint32_t (&w)[8], const PlaneLit& A,
                                           const PlaneLit& B, uint32_t& gtA, uint32_t& geA,
                                           uint32_t& gtB, uint32_t& geB) {
  gtA = bp_carry(w, A, 0u);
  geA = bp_carry(w, A, kFull);
  gtB = bp_carry(w, B, 0u);
  geB = bp_carry(w, B, kFull);
}
// "x >= t" for a host-prepared threshold.
__device__ __forceinline__ uint32_t bp_ge(const uint32_t (&w)[8], const PlaneThr& T) {
  return bp_carry(w, T.a, T.c0);
}

// Byte of row r from its block's 8 bit-plane words: the byte column r >> 3
// of words 0..3 and 4..7 gathered with PRMT, each byte's bit (r & 7) moved to
// bit 0, and the four 0/1 bytes of each half packed into a nibble with one
// multiply (bits 28..31 of x * (2^28 + 2^21 + 2^14 + 2^7); no carries, the
// other partial products land on distinct lower bits).
__device__ __forceinline__ uint32_t bp_byte(const uint32_t (&w)[8], int r) {
  const uint32_t c = (uint32_t)r >> 3;
  const uint32_t sel = c * 0x11u + 0x40u;  // [a.c, b.c] in the low half
  const uint32_t P = __byte_perm(__byte_perm(w[3], w[2], sel), __byte_perm(w[1], w[0], sel),
                                 0x5410u);  // [w3.c, w2.c, w1.c, w0.c]
  const uint32_t Q = __byte_perm(__byte_perm(w[7], w[6], sel), __byte_perm(w[5], w[4], sel),
                                 0x5410u);  // [w7.c, w6.c, w5.c, w4.c]
  const uint32_t sh = (uint32_t)r & 7u;
  const uint32_t M = 0x10204080u;
  const uint32_t hi = (((P >> sh) & 0x01010101u) * M) >> 24;  // bits 4..7: w3..w0
  const uint32_t lo = (((Q >> sh) & 0x01010101u) * M) >> 28;  // bits 0..3: w7..w4
  return (hi & 0xF0u) | lo;
}

// Byte of row r of a bit-plane block in global memory (one 32-byte sector).
// 256-bit load that allocates in L1: sectors several rows of one tile share
// (dense selections: ~12 selected deep rows per deep sector at 20 %).
__device__ __forceinline__ void ldg256_l1(const void* p, uint32_t (&w)[8]) {
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}
__device__ __forceinline__ uint32_t bp_row_byte_l1(const uint8_t* blk, int r) {
  uint32_t w[8];
  ldg256_l1(blk, w);
  return bp_byte(w, r);
}

__device__ __forceinline__ uint32_t bp_row_byte(const uint8_t* blk, int r) {
  uint32_t w[8];
  ldg256_free(blk, w);
  return bp_byte(w, r);
}
// ... and of a block staged in shared memory (16-byte aligned).
__device__ __forceinline__ uint32_t bp_row_byte_smem(const uint8_t* blk, int r) {
  const uint4 a = reinterpret_cast<const uint4*>(blk)[0];
  const uint4 b = reinterpret_cast<const uint4*>(blk)[1];
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  return bp_byte(w, r);
}

// Warp-cooperative write of one block of a plane: lane r holds row r's byte;
// lanes 0..7 store words 0..7 (one 32-byte sector).
__device__ __forceinline__ void bp_store_block(uint8_t* blk, uint32_t byte, int lane) {
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wk = __ballot_sync(kFull, (byte >> (7 - k)) & 1u);
    if (lane == k) mine = wk;
  }
  if (lane < 8) reinterpret_cast<uint32_t*>(blk)[lane] = mine;
}

// Round-1 byte-split literal constants, still used by the reference-packed
// deep runs (BSB_DEEP_PACKED, variable-length byte runs per block): adding
// (255 - L) to a byte in a 16-bit lane carries into bit 8 iff byte > L;
// adding (256 - L) carries iff byte >= L.
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

// pdep by 8-bit table lookups in shared memory: for every mask byte m the
// values pdep8(v, m), v < 2^popc(m), sit at pdep_off[m] + v (3^8 = 6561
// entries; pdep_off[m] = sum over m' < m of 2^popc(m')).  A 32-bit pdep is
// four byte lookups plus the running shift of x: ~20 integer ops and 8
// shared loads instead of the ~45 integer ops of the butterfly below -- the
// deep-space scan is ALU-bound, the shared-memory pipe is idle.
constexpr int kPdepTab = 6561;
struct PdepTables {
  uint16_t off[256];
  uint8_t val[kPdepTab + 7];
};
// Cooperative fill by a whole CTA (then __syncthreads).
__device__ __forceinline__ void pdep_tables_init(PdepTables& t) {
  for (int m = threadIdx.x; m < 256; m += blockDim.x) {
    uint32_t off = 0, p3 = 1;  // sum over set bits i of m: 2^popc(m >> (i+1)) * 3^i
    for (int i = 0; i < 8; ++i) {
      if ((m >> i) & 1) off += (1u << __popc((uint32_t)m >> (i + 1))) * p3;
      p3 *= 3;
    }
    t.off[m] = (uint16_t)off;
  }
  __syncthreads();
  for (int m = threadIdx.x >> 3; m < 256; m += blockDim.x >> 3) {
    const int nv = 1 << __popc((uint32_t)m);
    for (int v = threadIdx.x & 7; v < nv; v += 8) {
      uint32_t r = 0, k = 0;
      for (int i = 0; i < 8; ++i)
        if ((m >> i) & 1) r |= ((v >> k++) & 1u) << i;
      t.val[t.off[m] + v] = (uint8_t)r;
    }
  }
}
__device__ __forceinline__ uint32_t pdep_tab(const PdepTables& t, uint32_t x, uint32_t m) {
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t mb = (m >> (8 * b)) & 0xFFu;
    const uint32_t c = __popc(mb);
    r |= (uint32_t)t.val[t.off[mb] + (x & ((1u << c) - 1u))] << (8 * b);
    x >>= c;
  }
  return r;
}
// Same lookups from a global copy (read-only path: the 7 KB stay in L1).
__device__ __forceinline__ uint32_t pdep_tab_g(const PdepTables* t, uint32_t x, uint32_t m) {
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t mb = (m >> (8 * b)) & 0xFFu;
    const uint32_t c = __popc(mb);
    const uint32_t o = __ldg(t->off + mb);
    r |= (uint32_t)__ldg(t->val + o + (x & ((1u << c) - 1u))) << (8 * b);
    x >>= c;
  }
  return r;
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
