// bsb_vbs_ds.cu -- PP-VBS scan in deep-row space (SLICED layout).
//
// The reference's Alg. 3 (vbs.py:222-289) classifies each row by its own
// bytes only, so the rows split cleanly by code length:
//   * a row with a 1-byte code ("shallow", M_2 bit 0) is decided at level 1:
//     gt = byte > lit, eq_final = byte == lit only when the literal has one
//     byte (a shorter code tied on its own bytes is less, vbs.py:273-275);
//   * a row with a longer code ("deep") runs levels 1..len entirely on the
//     deep-row ByteSlice column: level-1 byte from deep[0] (or settled by the
//     column's zone map when all deep rows share their first byte), byte j
//     from deep[j-1], existence of byte j+1 from rexist[j] (byte 2 always
//     exists).
// Row space therefore needs no level-1 tie masks and no pext into deep-row
// order: phase 1 (lane = row block) computes the shallow rows' result and the
// block's deep-row offset; phase 2 (lane = deep block of the super-tile) runs
// Alg. 3 over the deep rows with early stop per deep block and writes one
// final-result word per deep block; phase 3 deposits each row block's window
// of deep results at its M_2 lanes (pdep) and writes the result word.
//
// The shallow rows' result is a function of two byte thresholds (host-chosen
// from the operator and the literals' first bytes).  L1 = false: no shallow
// row can match (e.g. a BETWEEN whose legs share their first byte with a
// multi-byte lo literal, or EQ with a multi-byte literal), so phase 1 reads
// only the M_2 words -- no first-slice bytes at all.
// The next super-tile's directory, M_2 words and level-1 deep sectors are
// requested across phases; the L1 variant prefetches the next super-tile's
// first-slice bytes into L2 (cp.async.bulk.prefetch) instead of holding them
// in registers.  Masked scans: EPI (this kernel) or vbs_dsm_kernel (below).
// Measured and dropped: L2 prefetch of deep levels, level j+1
// requested with level j, cp.async staging of deep levels in shared memory,
// 5-6 CTAs/SM, extra compare bodies (0x00 / adjacent literal bytes) -- the
// kernel is issue-bound and sensitive to code layout, not latency-bound.
#include <cstdlib>
#include <cstring>

#include "bsb_scan_impl.cuh"

namespace bsb {

constexpr int kDsThreads = 256;
constexpr int kDsWarps = kDsThreads / 32;

struct DsArgs {
  int64_t n_rows, nb, ntiles;
  int64_t full_tiles;
  int64_t nbpad;      // blocks covered by exist[1] / block_dir[1] (stride / 32)
  int serial_blocks;  // warp-cooperative pdep up to this many blocks per tile
  // Row-space level 1 (L1 variant): shallow result = valid & ~M_2 &
  // ((P & ~Q) ^ inv) with P = [byte >= tP], Q = [byte >= tQ] (bit-plane
  // thresholds, bsb_common.cuh); twoQ == 0 skips the Q compare (tQ = 256).
  PlaneThr tP, tQ;
  int twoQ;
  uint32_t inv;
  // Level 1 of the deep rows when they all share one first byte (zone map):
  // d1 = 1, and the per-leg (gt, eq) masks are constants (kFull or 0).
  int d1;
  uint32_t d1gA, d1eA, d1gB, d1eB;
  VbsDesc d;
  Leg A, B;
  const uint32_t* mask;  // input mask words (masked scans)
  uint32_t* out;
  unsigned long long* count;
  // running-mask gate (conjunction chains): *gate = the mask's row count;
  // the compacted kernel runs when it is <= gate_max, the EPI kernel otherwise
  const unsigned long long* gate;
  unsigned long long gate_max;
  const PdepTables* pdep;  // 8-bit pdep tables (g_pdep_tables, filled once)
};

__device__ PdepTables g_pdep_tables;

__global__ void pdep_tables_kernel() { pdep_tables_init(g_pdep_tables); }

// Fills the global pdep tables once per process (on the caller's stream, so
// a first call inside graph capture records the fill into the graph).
const PdepTables* pdep_tables(cudaStream_t s) {
  static const PdepTables* ptr = nullptr;
  if (!ptr) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_pdep_tables) != cudaSuccess) return nullptr;
    pdep_tables_kernel<<<1, 256, 0, s>>>();
    ptr = static_cast<const PdepTables*>(p);
  }
  return ptr;
}

__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// (gt, eq) of both legs at level index j0 (0-based) over a bit-plane block;
// legs with the same literal byte share one compare.
template <bool BETWEEN>
__device__ __forceinline__ void cmp_level(const uint32_t (&w)[8], const Leg& A, const Leg& B,
                                          int j0, uint32_t& gA, uint32_t& eA, uint32_t& gB,
                                          uint32_t& eB) {
  if (!BETWEEN || A.byte[j0] == B.byte[j0]) {
    uint32_t ge;
    cmp_block(w, A.pl[j0], gA, ge);
    eA = ge & ~gA;
    gB = gA;
    eB = eA;
  } else {
    uint32_t geA, geB;
    cmp_block2(w, A.pl[j0], B.pl[j0], gA, geA, gB, geB);
    eA = geA & ~gA;
    eB = geB & ~gB;
  }
}

__device__ __forceinline__ uint32_t lane_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// One Alg. 3 level over the lane's deep block (vbs.py:258-284 in deep-row
// space); false once no lane of the warp has a tied row left.
template <bool BETWEEN, bool DEADLEG, bool SPARSE = false>
__device__ __forceinline__ bool ds_level(const DsArgs& a, int j, int64_t dbk, const uint32_t* pre,
                                         uint32_t& zA, uint32_t& zB, uint32_t& gtA,
                                         uint32_t& eqA, uint32_t& gtB, uint32_t& eqB) {
  const VbsDesc& d = a.d;
  const int K = d.K;
  const bool act = BETWEEN ? ((zA | zB) != 0) : (zA != 0);
  if (!__any_sync(kFull, act)) return false;
  uint32_t w[8];
  if (j == 1 && pre != nullptr) {  // level-1 sector requested one phase earlier
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = pre[q];
  } else if (act) {
    if (j >= 3 || SPARSE)
      ldg256_sparse(d.deep[j - 1] + dbk * 32, w);  // only deep blocks still tied
    else
      ldg256(d.deep[j - 1] + dbk * 32, w);
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = 0;
  }
  // existence of byte j+1 among the deep rows (byte 2 always exists)
  const uint32_t nxt = j >= K ? 0u : (j == 1 ? kFull : (act ? __ldg(d.rexist[j] + dbk) : 0u));
  uint32_t gA, eA, gB, eB;
  if (BETWEEN && DEADLEG && a.A.byte[j - 1] != a.B.byte[j - 1]) {
    // a leg past its literal's last byte has no tied row left: no compare
    // (compiled into the L1 kernels only: the extra compare bodies cost the
    // other variants more than they save, measured)
    const bool liveA = j <= a.A.len, liveB = j <= a.B.len;
    if (liveA && liveB) {
      cmp_level<true>(w, a.A, a.B, j - 1, gA, eA, gB, eB);
    } else if (liveA) {
      cmp_level<false>(w, a.A, a.A, j - 1, gA, eA, gB, eB);
    } else {
      cmp_level<false>(w, a.B, a.B, j - 1, gB, eB, gA, eA);
    }
  } else {
    cmp_level<BETWEEN>(w, a.A, a.B, j - 1, gA, eA, gB, eB);
  }
  vbs_transition(j, a.A.len, K, gA, eA, nxt, zA, gtA, eqA);
  if (BETWEEN) {
    vbs_transition(j, a.B.len, K, gB, eB, nxt, zB, gtB, eqB);
    zB &= zA | gtA | eqA;  // hi-leg ties that already fail GE(lo) are settled
  }
  return true;
}

// EPI (masked scans with a dense mask): the column is scanned as if unmasked
// and the mask is AND-ed into the result words in phase 3 -- the same words
// (AND is idempotent).  With a gate, EPI runs when the mask's row count is
// above gate_max and the compacted vbs_dsm_kernel otherwise.
// LM: the shallow (1-byte-code) rows' result -- 0: none matches, 1: compared
// against the first-slice bytes (the "L1" code paths), 2: every one matches;
// 0 and 2 read no first-slice byte (constants of the literals).
template <bool BETWEEN, int LM, int ST, bool UNR, bool EPI = false>
__global__ void __launch_bounds__(kDsThreads, 4) vbs_ds_kernel(const __grid_constant__ DsArgs a) {
  constexpr bool L1 = LM == 1;
  if (EPI && a.gate && *a.gate <= a.gate_max) return;
  constexpr int kRd = ST * 32 + 8;  // deep blocks touched by a super-tile (+ guard)
  __shared__ uint32_t rd_all[kDsWarps][kRd];
  uint32_t* rd = rd_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VbsDesc& d = a.d;
  const int K = d.K;
  const Leg& A = a.A;
  const Leg& B = a.B;
  const int lenA = A.len, lenB = BETWEEN ? B.len : 0;
  const int maxlen = lenA > lenB ? lenA : lenB;
  const int64_t nsuper = (a.ntiles + ST - 1) / ST;
  unsigned long long cnt = 0;

  // level-1 sector (L1 only) and M_2 word of block b; zeros past the column
  auto fetch = [&](int64_t b, uint32_t (&w)[8], uint32_t& m2, bool bytes) {
    const bool in = b < a.nb;
    if (L1 && bytes) {
      if (in) {
        ldg256(d.bs1 + b * 32, w);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0;
      }
    }
    m2 = in ? __ldg(d.exist[1] + b) : 0u;
  };
  auto dir_at = [&](int64_t blk) -> int64_t {
    return __ldg(d.dir[1] + (blk < a.nbpad ? blk : a.nbpad));
  };

  // Software pipeline over this warp's super-tiles: the next super-tile's
  // directory bounds are requested at the top of an iteration, its M_2 words
  // and level-1 deep sectors right after phase 2, so that phase 3 and the
  // next phase 1 cover their latency.
  auto load_m2 = [&](int64_t s, uint32_t (&m)[ST], uint32_t (&mk)[ST]) {
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t b = (s * ST + u) * 32 + lane;
      m[u] = b < a.nb ? __ldg(d.exist[1] + b) : 0u;
      if (EPI) mk[u] = b < a.nb ? __ldg(a.mask + b) : 0u;
    }
  };
  auto load_l1 = [&](int64_t lo, int64_t hi, uint32_t (&w)[8]) {
    const int64_t dbk = (lo >> 5) + lane;
    if (dbk < ((hi + 31) >> 5)) {
      ldg256(d.deep[0] + dbk * 32, w);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = 0;
    }
  };

  int64_t st = warp;
  uint32_t m2P[ST], mP[ST], wP[8], wN[8];
  int64_t dlo = 0;
  if (st < nsuper) {
    dlo = dir_at(st * ST * 32);
    load_m2(st, m2P, mP);
    if (!L1 && !a.d1) load_l1(dlo, dir_at(st * ST * 32 + ST * 32), wP);
  }
  for (; st < nsuper; st += nwarps) {
    const int64_t sn = st + nwarps;
    const bool has_next = sn < nsuper;
    const int64_t nxt_b0 = sn * ST * 32;
    int64_t nlo = 0, nhi = 0;
    if (has_next) {
      nlo = dir_at(nxt_b0);
      if (!L1 && !a.d1) nhi = dir_at(nxt_b0 + ST * 32);
    }
    uint32_t rs[ST], m2s[ST], vs[ST];
    int offs[ST];
    int soff = 0;  // deep rows of this super-tile so far
    const int sh0 = (int)(dlo & 31);
    // first tile's bytes (L2-prefetched by the previous super-tile)
    if (L1) fetch(st * ST * 32 + lane, wN, m2s[0], true);
    // ---------------- phase 1: shallow rows (lane = row block)
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t tile = st * ST + u;
      const int64_t b = tile * 32 + lane;
      const uint32_t m2 = m2P[u];
      uint32_t valid =
          tile < a.full_tiles ? kFull : (tile < a.ntiles ? tail_valid(b, a.n_rows) : 0u);
      uint32_t res = LM == 2 ? (valid & ~m2) : 0u;
      if (L1) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = wN[i];
        uint32_t unused;
        if (u + 1 < ST) fetch(b + 32, wN, unused, true);
        const uint32_t P = bp_ge(w, a.tP);
        const uint32_t Q = a.twoQ ? bp_ge(w, a.tQ) : 0u;
        res = valid & ~m2 & ((P & ~Q) ^ a.inv);
      }
      rs[u] = res;
      m2s[u] = m2;
      if (EPI) vs[u] = mP[u];
      const int c2 = __popc(m2);
      const uint32_t incl = lane_incl_scan((uint32_t)c2, lane);
      offs[u] = soff + (int)(incl - (uint32_t)c2);
      soff += (int)__shfl_sync(kFull, incl, 31);
    }
    // next super-tile's first-slice bytes -> L2 (its first tile is loaded at
    // the top of the next iteration)
    if (L1 && has_next && lane == 0) {
      const int64_t nblk = a.nbpad - nxt_b0 < ST * 32 ? a.nbpad - nxt_b0 : ST * 32;
      l2_prefetch(d.bs1 + nxt_b0 * 32, (uint32_t)(nblk * 32));
    }
    // ---------------- phase 2: deep rows (lane = deep block)
    const int64_t db0 = dlo >> 5;
    const int ndt = (sh0 + soff + 31) >> 5;
    for (int t0 = 0; t0 < ndt; t0 += 32) {
      const int t = t0 + lane;
      const bool has = t < ndt;
      const int64_t dbk = db0 + t;
      // (the L1 variant's registers go to phase 1: no level-1 prefetch there)
      const uint32_t* pre = (!L1 && t0 == 0) ? wP : nullptr;
      const bool go = has;
      uint32_t zA = go ? kFull : 0u, zB = (BETWEEN && go) ? kFull : 0u;
      uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
      int j0 = 1;
      if (a.d1) {  // level 1 settled by the zone map: no deep[0] bytes read
        vbs_transition(1, A.len, K, a.d1gA, a.d1eA, kFull, zA, gtA, eqA);
        if (BETWEEN) {
          vbs_transition(1, B.len, K, a.d1gB, a.d1eB, kFull, zB, gtB, eqB);
          zB &= zA | gtA | eqA;
        }
        j0 = 2;
      }
      if (UNR) {
#pragma unroll
        for (int j = 1; j <= kMaxLevels; ++j) {
          if (j < j0) continue;
          if (j > maxlen ||
              !ds_level<BETWEEN, L1>(a, j, dbk, pre, zA, zB, gtA, eqA, gtB, eqB))
            break;
        }
      } else {
#pragma unroll 1
        for (int j = j0; j <= maxlen; ++j)
          if (!ds_level<BETWEEN, L1>(a, j, dbk, pre, zA, zB, gtA, eqA, gtB, eqB)) break;
      }
      if (has) rd[t] = BETWEEN ? ((gtA | eqA) & ~gtB) : finalize_op(A.op, gtA, eqA, kFull);
    }
    if (lane == 0) rd[ndt] = 0u;  // guard word of the last window
    if (has_next) {
      load_m2(sn, m2P, mP);
      if (!L1 && !a.d1) load_l1(nlo, nhi, wP);
    }
    dlo = nlo;
    __syncwarp();
    // ---------------- phase 3: deep results back to row space (lane = row block)
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t b = (st * ST + u) * 32 + lane;
      const uint32_t m2 = m2s[u];
      const int o = sh0 + offs[u];
      const int wi = o >> 5, sb = o & 31;
      const int c2 = __popc(m2);
      const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
      const uint32_t x = c2 ? (__funnelshift_r(rd[wi], rd[wi + 1], sb) & lowm) : 0u;
      uint32_t e = x ? m2 : 0u;
      const bool ntr = x != 0u && x != lowm;
      const uint32_t ntm = __ballot_sync(kFull, ntr);
      if (ntm) {
        if (__popc(ntm) > a.serial_blocks) {
          if (ntr) e = pdep_tab_g(a.pdep, x, m2);
        } else {
          for (uint32_t r = ntm; r; r &= r - 1) {
            const int L = __ffs(r) - 1;
            const uint32_t y =
                warp_pdep(__shfl_sync(kFull, m2, L), __shfl_sync(kFull, x, L), lane);
            if (lane == L) e = y;
          }
        }
      }
      const uint32_t res = EPI ? ((rs[u] | e) & vs[u]) : (rs[u] | e);
      if (b < a.nb) a.out[b] = res;
      cnt += __popc(res);
    }
    __syncwarp();
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

// 16-byte cp.async into shared memory, 64-byte DRAM fetch (sparse sectors).
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
// 16-byte cp.async of the first src_bytes (zero-filled after), dense stream.
__device__ __forceinline__ void cp_async16z(void* smem, const void* g, int src_bytes) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Masked scans with compacted work (conjunction legs under a sparse running
// mask, masked scan_vbs).  Same three phases as vbs_ds_kernel, but every
// phase runs over a per-warp list instead of lane = block:
//   * lists: lane = R consecutive row blocks of the super-tile (32 R blocks;
//     their M_2 / mask words staged one super-tile ahead by cp.async);
//     valid = tail & mask; one packed warp scan gives every block's deep-row
//     offset and its slot in L_1 (blocks with masked-in shallow rows: the
//     first-slice compare) and L_3 (blocks with masked-in deep rows: the
//     deposit); L_d (deep blocks holding L_3's rows) follows from L_3's
//     sorted deep-row ranges;
//   * L_1's first-slice sectors are staged in shared memory by cp.async
//     while phase 2 runs, so the two dependent chains overlap;
//   * phase 2 runs Alg. 3 over L_d only (lane = list entry), phase 1
//     compares the staged sectors, phase 3 deposits L_3's windows;
//   * each lane writes its R result words (zeros where the mask empties a
//     block; the same words as scanning whole and AND-ing the mask).
// Instructions and sectors scale with the masked-in blocks, not the column.
template <bool BETWEEN, int LM, int R, int WARPS, int MINB, int STAGE>
__global__ void __launch_bounds__(WARPS * 32, MINB) vbs_dsm_kernel(const __grid_constant__ DsArgs a) {
  constexpr bool L1 = LM == 1;
  if (a.gate && *a.gate > a.gate_max) return;
  static_assert(R == 4 || R == 8, "R row blocks per lane: 4 or 8");
  constexpr int NB = R * 32;    // row blocks per super-tile
  constexpr int kRd = NB + 8;   // deep blocks touched by a super-tile (+ guard)
  constexpr int kStage = L1 ? STAGE : 1;  // staged first-slice sectors per super-tile
  // packed scan fields: deep rows | L_1 entries | L_3 entries
  constexpr int kB1 = R == 4 ? 14 : 14, kB3 = R == 4 ? 23 : 23;
  struct __align__(16) Sm {
    uint32_t sec[kStage][8];
    uint32_t pm2[NB], pmk[NB];  // next super-tile's M_2 / mask words (cp.async)
    uint32_t res[NB], m2[NB], vw[NB], rd[kRd];
    uint16_t offs[NB], l1[NB], l3[NB], ld[kRd];
  };
  __shared__ Sm sm_all[WARPS];
  Sm& S = sm_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VbsDesc& d = a.d;
  const int K = d.K;
  const Leg& A = a.A;
  const Leg& B = a.B;
  const int lenA = A.len, lenB = BETWEEN ? B.len : 0;
  const int maxlen = lenA > lenB ? lenA : lenB;
  const int64_t nsuper = (a.nb + NB - 1) / NB;
  unsigned long long cnt = 0;
  auto dir_at = [&](int64_t blk) -> int64_t {
    return __ldg(d.dir[1] + (blk < a.nbpad ? blk : a.nbpad));
  };
  // M_2 and mask words of super-tile s -> pm2 / pmk (one commit group;
  // words past the column are zero-filled)
  auto stage_m2 = [&](int64_t s) {
#pragma unroll
    for (int c = lane; c < NB / 4; c += 32) {
      const int64_t w0 = s * NB + c * 4;
      const int64_t rem = a.nb - w0;
      const int nbytes = rem >= 4 ? 16 : (rem > 0 ? (int)rem * 4 : 0);
      cp_async16z(&S.pm2[c * 4], d.exist[1] + (nbytes ? w0 : 0), nbytes);
      cp_async16z(&S.pmk[c * 4], a.mask + (nbytes ? w0 : 0), nbytes);
    }
    cp_async_commit();
  };

  int64_t st = warp;
  int64_t dlo = 0;
  if (st < nsuper) {
    dlo = dir_at(st * NB);
    stage_m2(st);
  }
  for (; st < nsuper; st += nwarps) {
    const int64_t sn = st + nwarps;
    const bool has_next = sn < nsuper;
    const int64_t nlo = has_next ? dir_at(sn * NB) : 0;
    const int sh0 = (int)(dlo & 31);
    const int64_t b0 = st * NB + lane * R;  // this lane's first row block
    cp_async_wait_all();
    __syncwarp();
    // ---------------- lists (lane = R consecutive row blocks)
    uint32_t m[R], v[R];
#pragma unroll
    for (int q = 0; q < R; q += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(&S.pm2[lane * R + q]);
      const uint4 y = *reinterpret_cast<const uint4*>(&S.pmk[lane * R + q]);
      m[q] = x.x; m[q + 1] = x.y; m[q + 2] = x.z; m[q + 3] = x.w;
      v[q] = y.x; v[q + 1] = y.y; v[q + 2] = y.z; v[q + 3] = y.w;
    }
    if ((st + 1) * NB * 32 > a.n_rows) {  // last super-tile: rows past the column
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] &= b0 + r < a.nb ? tail_valid(b0 + r, a.n_rows) : 0u;
    }
    uint32_t tot = 0, f1 = 0, f3 = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      tot += __popc(m[r]);
      if (L1 && (v[r] & ~m[r])) f1 |= 1u << r;
      if (v[r] & m[r]) f3 |= 1u << r;
    }
    const uint32_t pk = tot | ((uint32_t)__popc(f1) << kB1) | ((uint32_t)__popc(f3) << kB3);
    const uint32_t incl = lane_incl_scan(pk, lane);
    const uint32_t all = __shfl_sync(kFull, incl, 31);
    const uint32_t ex = incl - pk;
    const int n1 = (int)((all >> kB1) & ((1u << (kB3 - kB1)) - 1u));
    const int n3 = (int)(all >> kB3);
    {
      int off = sh0 + (int)(ex & ((1u << kB1) - 1u));
      int p1 = (int)((ex >> kB1) & ((1u << (kB3 - kB1)) - 1u));
      int p3 = (int)(ex >> kB3);
      uint16_t o16[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint16_t i = (uint16_t)(lane * R + r);
        o16[r] = (uint16_t)off;
        off += __popc(m[r]);
        if ((f1 >> r) & 1u) S.l1[p1++] = i;
        if ((f3 >> r) & 1u) S.l3[p3++] = i;
      }
#pragma unroll
      for (int q = 0; q < R; q += 4) {
        *reinterpret_cast<uint4*>(&S.m2[lane * R + q]) = make_uint4(m[q], m[q + 1], m[q + 2], m[q + 3]);
        *reinterpret_cast<uint4*>(&S.vw[lane * R + q]) = make_uint4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        // shallow rows: compared in phase 1 (LM 1), else a constant of the literals
        *reinterpret_cast<uint4*>(&S.res[lane * R + q]) =
            LM == 2 ? make_uint4(v[q] & ~m[q], v[q + 1] & ~m[q + 1], v[q + 2] & ~m[q + 2],
                                 v[q + 3] & ~m[q + 3])
                    : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint2*>(&S.offs[lane * R + q]) =
            make_uint2((uint32_t)o16[q] | ((uint32_t)o16[q + 1] << 16),
                       (uint32_t)o16[q + 2] | ((uint32_t)o16[q + 3] << 16));
      }
    }
    __syncwarp();
    // first-slice sectors of L_1 -> shared memory (in flight during phase 2)
    if (L1) {
      const int ns = n1 < kStage ? n1 : kStage;
      for (int i = lane; i < ns; i += 32) {
        const uint8_t* g = d.bs1 + (st * NB + S.l1[i]) * 32;
        cp_async16(&S.sec[i][0], g);
        cp_async16(&S.sec[i][4], g + 16);
      }
      cp_async_commit();
    }
    // next super-tile's M_2 and mask words (always one group: wait_group 1
    // below then means "the first-slice sectors have landed")
    if (has_next) {
      stage_m2(sn);
    } else {
      cp_async_commit();
    }
    // L_d: deep blocks of L_3's rows.  L_3 is in block order, so its deep-row
    // ranges [lo, hi] (hi <= lo + 1) are sorted and meet only at endpoints.
    int nd = 0;
    {
      int prev_hi = -1;
      for (int k0 = 0; k0 < n3; k0 += 32) {
        const int k = k0 + lane;
        const bool has = k < n3;
        int lo = 0, hi = 0;
        if (has) {
          const int blk = S.l3[k];
          const int o = (int)S.offs[blk];
          lo = o >> 5;
          hi = (o + __popc(S.m2[blk]) - 1) >> 5;
        }
        int ph = __shfl_up_sync(kFull, hi, 1);
        if (lane == 0) ph = prev_hi;
        const bool e1 = has && lo != ph, e2 = has && hi != lo;
        const uint32_t b1 = __ballot_sync(kFull, e1), b2 = __ballot_sync(kFull, e2);
        const int pos = nd + __popc(b1 & lt) + __popc(b2 & lt);
        if (e1) S.ld[pos] = (uint16_t)lo;
        if (e2) S.ld[pos + (e1 ? 1 : 0)] = (uint16_t)hi;
        nd += __popc(b1) + __popc(b2);
        const int last = (n3 - k0 < 32 ? n3 - k0 : 32) - 1;
        prev_hi = __shfl_sync(kFull, hi, last);
      }
    }
    __syncwarp();
    // ---------------- phase 2: listed deep blocks (lane = list entry)
    const int64_t db0 = dlo >> 5;
    for (int t0 = 0; t0 < nd; t0 += 32) {
      const int i = t0 + lane;
      const bool has = i < nd;
      const int t = has ? (int)S.ld[i] : 0;
      const int64_t dbk = db0 + t;
      uint32_t zA = has ? kFull : 0u, zB = (BETWEEN && has) ? kFull : 0u;
      uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
      int j0 = 1;
      if (a.d1) {
        vbs_transition(1, A.len, K, a.d1gA, a.d1eA, kFull, zA, gtA, eqA);
        if (BETWEEN) {
          vbs_transition(1, B.len, K, a.d1gB, a.d1eB, kFull, zB, gtB, eqB);
          zB &= zA | gtA | eqA;
        }
        j0 = 2;
      }
#pragma unroll
      for (int j = 1; j <= kMaxLevels; ++j) {
        if (j < j0) continue;
        if (j > maxlen ||
            !ds_level<BETWEEN, L1, true>(a, j, dbk, nullptr, zA, zB, gtA, eqA, gtB, eqB))
          break;
      }
      if (has) S.rd[t] = BETWEEN ? ((gtA | eqA) & ~gtB) : finalize_op(A.op, gtA, eqA, kFull);
    }
    // ---------------- phase 1: shallow rows of L_1
    if (L1) {
      cp_async_wait1();
      __syncwarp();
      for (int i = lane; i < n1; i += 32) {
        const int blk = S.l1[i];
        uint32_t w[8];
        if (i < kStage) {
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = S.sec[i][q];
        } else {
          ldg256_sparse(d.bs1 + (st * NB + blk) * 32, w);
        }
        const uint32_t P = bp_ge(w, a.tP);
        const uint32_t Q = a.twoQ ? bp_ge(w, a.tQ) : 0u;
        S.res[blk] = S.vw[blk] & ~S.m2[blk] & ((P & ~Q) ^ a.inv);
      }
    }
    __syncwarp();
    // ---------------- phase 3: deep results of L_3 back to row space
    for (int i = lane; i < n3; i += 32) {
      const int blk = S.l3[i];
      const uint32_t m2 = S.m2[blk];
      const int o = (int)S.offs[blk];
      const int wi = o >> 5, sb = o & 31;
      const int c2 = __popc(m2);
      const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
      const uint32_t x = __funnelshift_r(S.rd[wi], S.rd[wi + 1], sb) & lowm;
      const uint32_t e = x == 0u ? 0u : (x == lowm ? m2 : pdep_tab_g(a.pdep, x, m2));
      S.res[blk] |= e & S.vw[blk];
    }
    __syncwarp();
    // ---------------- result words (lane = its R row blocks)
#pragma unroll
    for (int q = 0; q < R; q += 4) {
      const uint4 r4 = *reinterpret_cast<const uint4*>(&S.res[lane * R + q]);
      cnt += __popc(r4.x) + __popc(r4.y) + __popc(r4.z) + __popc(r4.w);
      if (b0 + q + 4 <= a.nb) {
        *reinterpret_cast<uint4*>(a.out + b0 + q) = r4;
      } else {
        const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (b0 + q + e < a.nb) a.out[b0 + q + e] = rr[e];
      }
    }
    dlo = nlo;
    __syncwarp();
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

template <bool BETWEEN, int LM, int R, int WARPS, int MINB, int STAGE>
static int launch_dsm_k(const DsArgs& a, cudaStream_t s) {
  auto kern = vbs_dsm_kernel<BETWEEN, LM, R, WARPS, MINB, STAGE>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, 0);
  if (per_sm < 1) per_sm = 1;
  if (ctas_per_sm_cap() > 0 && per_sm > ctas_per_sm_cap()) per_sm = ctas_per_sm_cap();
  const int64_t nsuper = (a.nb + R * 32 - 1) / (R * 32);
  const int64_t want = (nsuper + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  kern<<<grid, WARPS * 32, 0, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}
static int tune(int i);
template <bool BETWEEN, int LM>
static int launch_dsm(const DsArgs& a, cudaStream_t s) {
  switch (tune(6)) {
    case 1: return launch_dsm_k<BETWEEN, LM, 4, 8, 6, 16>(a, s);
    case 2: return launch_dsm_k<BETWEEN, LM, 8, 4, 6, 32>(a, s);
    case 3: return launch_dsm_k<BETWEEN, LM, 8, 4, 4, 64>(a, s);
    default: return launch_dsm_k<BETWEEN, LM, 4, 8, 4, 32>(a, s);
  }
}

template <bool BETWEEN, int LM, int ST, bool UNR, bool EPI = false>
static int launch_ds_k(const DsArgs& a, cudaStream_t s) {
  auto kern = vbs_ds_kernel<BETWEEN, LM, ST, UNR, EPI>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDsThreads, 0);
  if (per_sm < 1) per_sm = 1;
  if (ctas_per_sm_cap() > 0 && per_sm > ctas_per_sm_cap()) per_sm = ctas_per_sm_cap();
  const int64_t nsuper = (a.ntiles + ST - 1) / ST;
  const int64_t want = (nsuper + kDsWarps - 1) / kDsWarps;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  kern<<<grid, kDsThreads, 0, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

template <bool BETWEEN, int LM, bool UNR>
static int launch_ds_u(const DsArgs& a, int st, cudaStream_t s) {
  switch (st) {
    case 1: return launch_ds_k<BETWEEN, LM, 1, UNR>(a, s);
    case 2: return launch_ds_k<BETWEEN, LM, 2, UNR>(a, s);
    case 3: return launch_ds_k<BETWEEN, LM, 3, UNR>(a, s);
    default: return launch_ds_k<BETWEEN, LM, 4, UNR>(a, s);
  }
}
template <bool BETWEEN, int LM>
static int launch_ds_epi(const DsArgs& a, int st, cudaStream_t s) {
  switch (st) {
    case 1: return launch_ds_k<BETWEEN, LM, 1, true, true>(a, s);
    case 2: return launch_ds_k<BETWEEN, LM, 2, true, true>(a, s);
    case 3: return launch_ds_k<BETWEEN, LM, 3, true, true>(a, s);
    default: return launch_ds_k<BETWEEN, LM, 4, true, true>(a, s);
  }
}
template <bool BETWEEN, int LM>
static int launch_ds(const DsArgs& a, int st, bool unr, cudaStream_t s) {
  if (!a.mask)
    return unr ? launch_ds_u<BETWEEN, LM, true>(a, st, s) : launch_ds_u<BETWEEN, LM, false>(a, st, s);
  // Masked: the compacted kernel and EPI behind the gate (the mask's row
  // count vs gate_max; each exits at once when the other applies), or EPI
  // alone when there is no gate, the gate is off (gate_max 0), bsb_tune
  // ds_masked=1, or a word array is not 16-byte aligned (the compacted kernel
  // moves M_2 / mask / result words 16 bytes at a time).
  const bool al16 = (((uintptr_t)a.mask | (uintptr_t)a.d.exist[1] | (uintptr_t)a.out) & 15u) == 0;
  if (!a.gate || a.gate_max == 0 || tune(5) != 0 || !al16) {
    DsArgs e = a;
    e.gate = nullptr;
    return launch_ds_epi<BETWEEN, LM>(e, st, s);
  }
  const int rc = launch_dsm<BETWEEN, LM>(a, s);
  return rc ? rc : launch_ds_epi<BETWEEN, LM>(a, st, s);
}

// Run-time tunables (bsb_tune): 0 enable (0 off, 1 all scans, 2 unmasked
// only), 1 serial pdep blocks, 2 tiles per super-tile (0 = auto), 3 unrolled
// levels, 4 settle the deep rows' level 1 from the column's zone map (0/1),
// 5 masked scans (0 gated compacted / EPI pair, 1 EPI only), 6 compacted
// kernel shape (rows blocks per lane, warps, CTAs per SM; see launch_dsm).
constexpr int kTunes = 7;
static int g_tune[kTunes] = {-1, -1, -1, -1, -1, -1, -1};
static const char* const kTuneKeys[kTunes] = {"ds_enable", "ds_serial", "ds_tiles", "ds_unroll",
                                              "ds_zonemap", "ds_masked", "dsm_cfg"};
static int tune(int i) {
  if (g_tune[i] < 0) {
    static const char* const env[kTunes] = {"BSB_DS", "BSB_DS_SERIAL", "BSB_DS_TILES",
                                            "BSB_DS_UNROLL", "BSB_DS_ZONEMAP", "BSB_DS_MASKED",
                                            "BSB_DSM_CFG"};
    static const int dflt[kTunes] = {1, 3, 0, 1, 1, 0, 0};
    const char* e = std::getenv(env[i]);
    g_tune[i] = e ? std::atoi(e) : dflt[i];
  }
  return g_tune[i];
}
// ds_enable: 0 off, 1 all scans, 2 unmasked scans only
bool ds_enabled(bool masked) { return masked ? tune(0) == 1 : tune(0) != 0; }
bool ds_zonemap_enabled() { return tune(4) != 0; }


// Shallow rows (vbs.py:272-284 with M_2 = 0): gt = byte > lit, eq_final =
// byte == lit only for a 1-byte literal, so the result of a 1-byte-code row
// is ([byte >= tP] & ~[byte >= tQ]) ^ inv with thresholds per operator (tQ =
// 256: no Q compare).  For BETWEEN, [byte >= tP] is exactly GE(lo).
void shallow_thresholds(const Leg& A, const Leg& B, bool between, int& tP, int& tQ,
                        uint32_t& inv) {
  const int la = (int)A.byte[0], lb = (int)B.byte[0];
  const int ge_a = la + (A.len >= 2 ? 1 : 0);  // [byte >= ge_a] == gt | eq_final
  tP = 256;
  tQ = 256;
  inv = 0;
  if (between) {
    tP = ge_a;
    tQ = lb + 1;
  } else {
    switch (A.op) {
      case BSB_GT: tP = la + 1; break;
      case BSB_GE: tP = ge_a; break;
      case BSB_LT: tP = ge_a; inv = kFull; break;
      case BSB_LE: tP = la + 1; inv = kFull; break;
      case BSB_EQ:
        if (A.len == 1) { tP = la; tQ = la + 1; }
        break;
      default:  // NE
        if (A.len == 1) { tP = la; tQ = la + 1; }
        inv = kFull;
        break;
    }
  }
}

// Scan of a SLICED column that carries deep[0] (K >= 2), optionally masked.
int vbs_ds_scan(const VbsDesc& d, int64_t n_rows, int64_t stride, int64_t deep_rows,
                int deep1_shared, const Leg& A, const Leg& B, bool between,
                const uint32_t* mask, uint32_t* out, unsigned long long* count,
                cudaStream_t s, const unsigned long long* gate,
                unsigned long long gate_max) {
  DsArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = n_rows;
  a.nb = (n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  a.full_tiles = n_rows / kTileRows;
  a.nbpad = stride / 32;
  const int st_env = tune(2);
  const bool unr = tune(3) != 0;
  a.serial_blocks = tune(1);
  a.d = d;
  a.A = A;
  a.B = B;
  a.mask = mask;
  a.out = out;
  a.count = count;
  a.gate = gate;
  a.gate_max = gate_max;
  a.pdep = pdep_tables(s);
  if (!a.pdep) return BSB_ECUDA;
  if (deep1_shared >= 1 && deep1_shared <= 256 && tune(4)) {
    const uint32_t x = (uint32_t)(deep1_shared - 1);
    a.d1 = 1;
    a.d1gA = x > A.byte[0] ? kFull : 0u;
    a.d1eA = x == A.byte[0] ? kFull : 0u;
    a.d1gB = x > B.byte[0] ? kFull : 0u;
    a.d1eB = x == B.byte[0] ? kFull : 0u;
  }
  // tiles per super-tile: about 28 deep blocks per phase-2 pass
  int st = st_env;
  if (st < 1 || st > 4) {
    const double per_tile = 32.0 * (double)deep_rows / (double)(n_rows > 0 ? n_rows : 1);
    st = per_tile > 0 ? (int)(28.0 / per_tile + 0.5) : 4;
    st = st < 1 ? 1 : (st > 4 ? 4 : st);
  }
  int tP, tQ;
  uint32_t inv;
  shallow_thresholds(A, B, between, tP, tQ, inv);
  a.tP = make_plane_thr(tP);
  a.tQ = make_plane_thr(tQ);
  a.twoQ = tQ < 256;
  a.inv = inv;
  // The shallow result ([byte >= tP] & ~[byte >= tQ]) ^ inv is a constant of
  // the literals when neither threshold can split a byte (tP, tQ outside
  // 1..255) or the window is empty: then no first-slice byte is read.  E.g.
  // LE / LT with a literal whose first byte is 255 (a value right of every
  // first-level slot: all of a Zipf column's long codes) matches every
  // 1-byte-code row; GE / GT / BETWEEN from such a value match none.
  const bool p_var = tP >= 1 && tP <= 255, q_var = tQ >= 1 && tQ <= 255;
  int lm = 1;
  if (!p_var && !q_var) {
    const bool pq = tP <= 0 && tQ >= 256;  // P always, Q never
    lm = (((pq ? kFull : 0u) ^ inv) != 0u) ? 2 : 0;
  } else if (!inv && tP >= tQ) {  // empty window
    lm = 0;
  }
  if (!gate) BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));  // gated: zeroed by the caller
  if (between) {
    switch (lm) {
      case 0: return launch_ds<true, 0>(a, st, unr, s);
      case 2: return launch_ds<true, 2>(a, st, unr, s);
      default: return launch_ds<true, 1>(a, st, unr, s);
    }
  }
  switch (lm) {
    case 0: return launch_ds<false, 0>(a, st, unr, s);
    case 2: return launch_ds<false, 2>(a, st, unr, s);
    default: return launch_ds<false, 1>(a, st, unr, s);
  }
}

}  // namespace bsb

namespace bsb {
void set_sparse_ppm(int64_t ppm);  // bsb_scan.cu
void set_conj_fuse(int64_t v);     // bsb_scan.cu
void set_ctas_per_sm_cap(int v);   // bsb_build.cu
void set_stats_rows(int64_t v);    // bsb_scan.cu
void set_scan_nomemset(int64_t v); // bsb_scan.cu
void set_bs_small(int64_t v);      // bsb_scan.cu
void set_pdl(int64_t v);           // bsb_scan.cu
void set_pair_bits(int64_t v);     // bsb_gather.cu
void set_coop_tiles(int64_t v);    // bsb_lookup.cu
void set_dense_rows(int64_t v);    // bsb_lookup.cu
}

extern "C" int bsb_tune(const char* key, int64_t value) {
  if (!key) return BSB_EINVAL;
  if (std::strcmp(key, "sparse_ppm") == 0) {  // sparse-mask gate, parts per million
    bsb::set_sparse_ppm(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "stats_rows") == 0) {  // PP-VBS ScanStats via the row kernel
    bsb::set_stats_rows(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "pdl") == 0) {  // programmatic dependent launch (0/1)
    bsb::set_pdl(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "bs_small") == 0) {  // small-column ByteSlice kernel (0/1)
    bsb::set_bs_small(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "scan_nomemset") == 0) {  // diagnostics: ByteSlice count not zeroed
    bsb::set_scan_nomemset(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "ctas_per_sm") == 0) {  // persistent-grid cap (0 = none)
    bsb::set_ctas_per_sm_cap((int)value);
    return BSB_OK;
  }
  if (std::strcmp(key, "dense_rows") == 0) {  // fused PP-VBS lookup: L1-allocating deep loads from
    bsb::set_dense_rows(value);               // this many selected rows per tile
    return BSB_OK;
  }
  if (std::strcmp(key, "coop_tiles") == 0) {  // one-kernel fused lookup up to this many tiles
    bsb::set_coop_tiles(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "pair_bits") == 0) {  // row buckets of bsb_rows_bucket (2^bits)
    bsb::set_pair_bits(value);
    return BSB_OK;
  }
  if (std::strcmp(key, "conj_fuse") == 0) {  // fused ByteSlice pairs in bsb_conj_scan
    bsb::set_conj_fuse(value);
    return BSB_OK;
  }
  for (int i = 0; i < bsb::kTunes; ++i)
    if (std::strcmp(key, bsb::kTuneKeys[i]) == 0) {
      bsb::g_tune[i] = value < 0 ? -1 : (int)value;  // < 0: back to the default
      return BSB_OK;
    }
  return BSB_EINVAL;
}
