// bsb_vbs_sliced.cu -- PP-VBS scan for the SLICED deep layout, three tiles
// per warp iteration.
//
// Phase 1 (lane = row block, one tile after another): level 1 with the SWAR
// compare on the prefetched first-slice sector and the reference transitions
// (vbs.py:258-284); the tied rows of each block are compressed into deep-row
// order (one butterfly set-up per block) and OR-ed into per-deep-block
// candidate words; the block's level-1 state and butterfly masks go to shared
// memory.
// Phase 2 (lane = deep block): the super-tile's deep rows form ~27 deep
// blocks for the cfg2 column, so the warp runs Alg. 3 levels 2..len over them
// at ~85% lane utilisation: one 256-bit load + SWAR compare per live deep
// block per level, early stop per deep block, transitions with the deep-row
// existence words.
// Phase 3 (lane = row block): each block expands its window of the deep
// results back to row space, finalises the operator and writes its word.
#include <cstdlib>
#include <cstring>

#include "bsb_scan_impl.cuh"

namespace bsb {

// Tiles per warp iteration (ST) is a template argument chosen per column so
// that a super-tile's deep rows fill about one warp of deep blocks.
template <int ST>
struct SuperTile {
  static constexpr int kTiles = ST;
  static constexpr int kBlocks = ST * 32;           // row blocks per iteration
  static constexpr int kMaxDeepBlocks = ST * 32 + 4;  // deep blocks touched (+ guard)
};
constexpr int kSlicedThreads = 256;
constexpr int kSlicedWarps = kSlicedThreads / 32;
// up to this many blocks with non-trivial masks per tile are compressed /
// expanded warp-cooperatively; more switch to the per-lane butterfly
constexpr int kSerialBlocks = 6;

struct SlicedArgs {
  int64_t n_rows, nb, ntiles;
  int64_t full_tiles;  // tiles whose 1024 rows are all < n_rows
  int serial_blocks;   // warp-cooperative pext/pdep up to this many blocks
  VbsDesc d;
  Leg A, B;
  const uint32_t* mask;
  uint32_t* out;
  unsigned long long* count;
};

template <int ST>
struct SlicedSmem {
  static constexpr int NB = SuperTile<ST>::kBlocks, ND = SuperTile<ST>::kMaxDeepBlocks;
  // per row block: level-1 state
  uint32_t valid[NB], zgtA[NB], eqfA[NB], zeqA[NB];
  uint32_t zgtB[NB], zeqB[NB], m2[NB], off[NB];
  // per deep block: candidates in, results out
  uint32_t cA[ND], cB[ND], rP[ND], rQ[ND];
};

template <bool BETWEEN, bool MASKED, int MINB, int ST>
__global__ void __launch_bounds__(kSlicedThreads, MINB)
    vbs_sliced_kernel(const __grid_constant__ SlicedArgs a) {
  constexpr int kSuperTiles = SuperTile<ST>::kTiles;
  constexpr int kMaxDeepBlocks = SuperTile<ST>::kMaxDeepBlocks;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SlicedSmem<ST>& sm = reinterpret_cast<SlicedSmem<ST>*>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VbsDesc& d = a.d;
  const int K = d.K;
  const Leg& A = a.A;
  const Leg& B = a.B;
  const int lenA = A.len, lenB = BETWEEN ? B.len : 0;
  const int maxlen = lenA > lenB ? lenA : lenB;
  const int64_t nsuper = (a.ntiles + kSuperTiles - 1) / kSuperTiles;
  unsigned long long cnt = 0;

  // valid rows of block b of tile t (input mask applied); 0 past the column
  auto tile_valid_word = [&](int64_t tile, int64_t b) -> uint32_t {
    uint32_t v = tile < a.full_tiles ? kFull : (tile < a.ntiles ? tail_valid(b, a.n_rows) : 0u);
    if (MASKED) v &= b < a.nb ? __ldg(a.mask + b) : 0u;
    return v;
  };
  // level-1 sector + level-2 existence word of block b (zeros when invalid)
  auto fetch = [&](int64_t b, uint32_t valid, TileIn& t) {
    if (valid) {
      ldg256(d.bs1 + b * 32, t.w);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) t.w[i] = 0;
    }
    t.m2 = (K >= 2 && b < a.nb) ? __ldg(d.exist[1] + b) : 0u;
  };

  // prefetch pipeline over the flattened tile sequence of this warp
  int64_t st = warp;
  TileIn inN;
  uint32_t vN = 0;
  if (st < nsuper) {
    const int64_t b0 = st * kSuperTiles * 32 + lane;
    vN = tile_valid_word(st * kSuperTiles, b0);
    fetch(b0, vN, inN);
  }
  for (; st < nsuper; st += nwarps) {
    // global deep row of the super-tile's first deep row
    const int64_t dfirst = K >= 2 ? __ldg(d.dir[1] + st * kSuperTiles * 32) : 0;
    const int64_t db0 = dfirst >> 5;
    int soff = (int)(dfirst & 31);  // running deep-row offset from db0 * 32
    for (int k = lane; k < kMaxDeepBlocks; k += 32) {
      sm.cA[k] = 0;
      sm.cB[k] = 0;
    }
    // ---------------- phase 1: level 1, three tiles
#pragma unroll
    for (int u = 0; u < kSuperTiles; ++u) {
      const int64_t tile = st * kSuperTiles + u;
      const uint32_t valid = vN;
      const TileIn in = inN;
      // prefetch the next tile in this warp's sequence
      const int64_t ntile = (u + 1 < kSuperTiles) ? tile + 1 : (st + nwarps) * kSuperTiles;
      const int64_t nb_ = ntile * 32 + lane;
      vN = tile_valid_word(ntile, nb_);
      fetch(nb_, vN, inN);
      uint32_t zeqA = valid, zgtA = 0, eqfA = 0, zeqB = valid, zgtB = 0, eqfB = 0;
      int depth = 0;
      vbs_level1<BETWEEN, false>(A, B, K, valid, in, zeqA, zgtA, eqfA, zeqB, zgtB, eqfB,
                                 nullptr, depth);
      const int c2 = __popc(in.m2);
      const uint32_t incl = warp_incl_scan((uint32_t)c2);
      const int o = soff + (int)(incl - (uint32_t)c2);
      // Tied rows -> deep-row order (pext by M_2).  zeq is a subset of M_2, so
      // zeq == 0 or zeq == M_2 compress trivially; the few other blocks of the
      // tile are compressed by the whole warp one at a time, or, when there are
      // many, by each lane's butterfly network (whose masks phase 3 reuses).
      const int i = u * 32 + lane;
      const uint32_t full = c2 >= 32 ? kFull : ((1u << c2) - 1u);
      uint32_t pA = zeqA ? full : 0u;
      uint32_t pB = (BETWEEN && zeqB) ? full : 0u;
      const bool ntr = (zeqA != 0 && zeqA != in.m2) || (BETWEEN && zeqB != 0 && zeqB != in.m2);
      uint32_t ntm = __ballot_sync(kFull, ntr);
      if (__popc(ntm) > a.serial_blocks) {
        const ExpandNet net = expand_setup(in.m2);
        pA = compress_apply(net, zeqA);
        if (BETWEEN) pB = compress_apply(net, zeqB);
      } else {
        while (ntm) {
          const int L = __ffs(ntm) - 1;
          ntm &= ntm - 1;
          const uint32_t mL = __shfl_sync(kFull, in.m2, L);
          const uint32_t x = warp_pext(mL, __shfl_sync(kFull, zeqA, L), lane);
          const uint32_t y = BETWEEN ? warp_pext(mL, __shfl_sync(kFull, zeqB, L), lane) : 0u;
          if (lane == L) {
            pA = x;
            pB = y;
          }
        }
      }
      sm.valid[i] = valid;
      sm.zgtA[i] = zgtA;
      sm.eqfA[i] = eqfA;
      sm.zeqA[i] = zeqA;
      sm.zgtB[i] = zgtB;
      sm.zeqB[i] = zeqB;
      sm.m2[i] = in.m2;
      sm.off[i] = (uint32_t)o;
      __syncwarp();
      const int wi = o >> 5, sb = o & 31;
      const bool spill = sb != 0 && sb + c2 > 32;
      if (pA && wi < kMaxDeepBlocks) {
        atomicOr(&sm.cA[wi], pA << sb);
        if (spill && wi + 1 < kMaxDeepBlocks) atomicOr(&sm.cA[wi + 1], pA >> (32 - sb));
      }
      if (BETWEEN && pB && wi < kMaxDeepBlocks) {
        atomicOr(&sm.cB[wi], pB << sb);
        if (spill && wi + 1 < kMaxDeepBlocks) atomicOr(&sm.cB[wi + 1], pB >> (32 - sb));
      }
      soff += (int)__shfl_sync(kFull, incl, 31);
    }
    __syncwarp();
    // ---------------- phase 2: deep blocks, one per lane
    const int ndt = (soff + 31) >> 5;
    if (maxlen >= 2) {
      for (int t0 = 0; t0 < ndt; t0 += 32) {
        const int t = t0 + lane;
        const bool has = t < ndt && t < kMaxDeepBlocks;
        uint32_t zA = has ? sm.cA[t] : 0u, zB = (BETWEEN && has) ? sm.cB[t] : 0u;
        uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
        const int64_t dbk = db0 + t;
        for (int j = 2; j <= maxlen; ++j) {
          const bool act = BETWEEN ? ((zA | zB) != 0) : (zA != 0);
          if (!__any_sync(kFull, act)) break;
          uint32_t w[8];
          if (act) {
            ldg256(d.deep[j - 1] + dbk * 32, w);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = 0;
          }
          const uint32_t nxt = (j < K && act) ? __ldg(d.rexist[j] + dbk) : 0u;
          uint32_t gA, eA, gB, eB;
          if (BETWEEN && A.byte[j - 1] != B.byte[j - 1]) {
            cmp_block2(w, A.pl[j - 1], B.pl[j - 1], gA, eA, gB, eB);
          } else {
            cmp_block(w, A.pl[j - 1], gA, eA);
            gB = gA;
            eB = eA;
          }
          eA &= ~gA;
          eB &= ~gB;
          vbs_transition(j, lenA, K, gA, eA, nxt, zA, gtA, eqA);
          if (BETWEEN) vbs_transition(j, lenB, K, gB, eB, nxt, zB, gtB, eqB);
        }
        if (has) {
          sm.rP[t] = BETWEEN ? (gtA | eqA) : gtA;
          sm.rQ[t] = BETWEEN ? gtB : eqA;
        }
      }
    }
    for (int k = ndt + lane; k < kMaxDeepBlocks; k += 32) {
      sm.rP[k] = 0;
      sm.rQ[k] = 0;
    }
    __syncwarp();
    // ---------------- phase 3: back to row space
#pragma unroll 1
    for (int u = 0; u < kSuperTiles; ++u) {
      const int64_t tile = st * kSuperTiles + u;
      if (tile >= a.ntiles) break;
      const int64_t b = tile * 32 + lane;
      const int i = u * 32 + lane;
      const uint32_t valid = sm.valid[i];
      uint32_t zgtA = sm.zgtA[i], eqfA = sm.eqfA[i], zgtB = sm.zgtB[i];
      const uint32_t zeqA = sm.zeqA[i], zeqB = sm.zeqB[i];
      if (maxlen >= 2) {
        const uint32_t m2 = sm.m2[i];
        const int o = (int)sm.off[i];
        const int c2 = __popc(m2);
        const int wi = o >> 5, sb = o & 31;
        const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
        uint32_t pP = 0, pQ = 0;
        if (wi + 1 < kMaxDeepBlocks) {
          pP = __funnelshift_r(sm.rP[wi], sm.rP[wi + 1], sb) & lowm;
          pQ = __funnelshift_r(sm.rQ[wi], sm.rQ[wi + 1], sb) & lowm;
        }
        // deep-row results -> row space (pdep by M_2).  A fused BETWEEN whose
        // two legs tie on the same rows (the common case: the literals share
        // their first byte) needs only the combined word "passes lo and not
        // above hi" -- one pdep, and trivial (all or nothing) for most
        // blocks of a selective window.
        const bool same = BETWEEN && zeqA == zeqB;
        const uint32_t x1 = same ? (pP & ~pQ) : pP;
        const uint32_t x2 = same ? 0u : pQ;
        uint32_t e1 = x1 ? m2 : 0u, e2 = x2 ? m2 : 0u;
        const uint32_t nt1 = __ballot_sync(kFull, x1 != 0 && x1 != lowm);
        const uint32_t nt2 = __ballot_sync(kFull, x2 != 0 && x2 != lowm);
        if (nt1 | nt2) {
          if (__popc(nt1 | nt2) > a.serial_blocks) {
            const ExpandNet net = expand_setup(m2);
            e1 = expand_apply(net, x1);
            e2 = expand_apply(net, x2);
          } else {
            for (uint32_t ntm = nt1; ntm; ntm &= ntm - 1) {
              const int L = __ffs(ntm) - 1;
              const uint32_t x = warp_pdep(__shfl_sync(kFull, m2, L),
                                           __shfl_sync(kFull, x1, L), lane);
              if (lane == L) e1 = x;
            }
            for (uint32_t ntm = nt2; ntm; ntm &= ntm - 1) {
              const int L = __ffs(ntm) - 1;
              const uint32_t x = warp_pdep(__shfl_sync(kFull, m2, L),
                                           __shfl_sync(kFull, x2, L), lane);
              if (lane == L) e2 = x;
            }
          }
        }
        if (same) {
          // tied rows take the deep verdict; the rest were decided at level 1
          const uint32_t l1 = (zgtA | eqfA) & ~zgtB;
          zgtA = (l1 & ~zeqA) | (e1 & zeqA);
          eqfA = 0u;
          zgtB = 0u;
        } else if (BETWEEN) {
          zgtA |= zeqA & e1;
          zgtB |= zeqB & e2;
        } else {
          zgtA |= zeqA & e1;
          eqfA |= zeqA & e2;
        }
      }
      const uint32_t res = BETWEEN ? (valid & (zgtA | eqfA) & ~zgtB)
                                   : finalize_op(A.op, zgtA, eqfA, valid);
      if (b < a.nb) a.out[b] = res;
      cnt += __popc(res);
    }
    __syncwarp();
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

template <bool BETWEEN, bool MASKED, int MINB, int ST>
static int launch_sliced_k(const SlicedArgs& a, cudaStream_t s) {
  constexpr int kSuperTiles = ST;
  auto kern = vbs_sliced_kernel<BETWEEN, MASKED, MINB, ST>;
  const size_t smem = sizeof(SlicedSmem<ST>) * kSlicedWarps;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSlicedThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t nsuper = (a.ntiles + kSuperTiles - 1) / kSuperTiles;
  int64_t want = (nsuper + kSlicedWarps - 1) / kSlicedWarps;
  int64_t cap = (int64_t)sm_count() * per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  kern<<<grid, kSlicedThreads, smem, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

// Occupancy variant: 4 resident CTAs (64 registers) by default;
// BSB_SLICED_MINB=3 selects the 80-register build (tuning experiments).
template <bool BETWEEN, bool MASKED>
static int launch_sliced(const SlicedArgs& a, int64_t deep_rows, cudaStream_t s) {
  static int minb = -1, st_env = -1;
  if (minb < 0) {
    const char* e = std::getenv("BSB_SLICED_MINB");
    minb = (e && std::atoi(e) == 3) ? 3 : 4;
    const char* t = std::getenv("BSB_SLICED_TILES");
    st_env = t ? std::atoi(t) : 0;
  }
  // tiles per super-tile: about 28 deep blocks (of 32 lanes) per phase 2
  int st = st_env;
  if (st < 1 || st > 4) {
    const double per_tile = 32.0 * (double)deep_rows / (double)(a.n_rows > 0 ? a.n_rows : 1);
    st = per_tile > 0 ? (int)(28.0 / per_tile + 0.5) : 4;
    st = st < 1 ? 1 : (st > 4 ? 4 : st);
  }
  if (minb == 3) return launch_sliced_k<BETWEEN, MASKED, 3, 3>(a, s);
  switch (st) {
    case 1: return launch_sliced_k<BETWEEN, MASKED, 4, 1>(a, s);
    case 2: return launch_sliced_k<BETWEEN, MASKED, 4, 2>(a, s);
    case 3: return launch_sliced_k<BETWEEN, MASKED, 4, 3>(a, s);
    default: return launch_sliced_k<BETWEEN, MASKED, 4, 4>(a, s);
  }
}

// Non-stats scan of a SLICED column (BETWEEN fused).  Legs as in ScanArgs.
int vbs_sliced_scan(const VbsDesc& d, int64_t n_rows, int64_t deep_rows, const Leg& A,
                    const Leg& B, bool between,
                    const uint32_t* mask, uint32_t* out, unsigned long long* count,
                    cudaStream_t s) {
  SlicedArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = n_rows;
  a.nb = (n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  a.full_tiles = n_rows / kTileRows;
  static int serial = -1;
  if (serial < 0) {
    const char* e = std::getenv("BSB_SLICED_SERIAL");
    serial = e ? std::atoi(e) : kSerialBlocks;
  }
  a.serial_blocks = serial;
  a.d = d;
  a.A = A;
  a.B = B;
  a.mask = mask;
  a.out = out;
  a.count = count;
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  if (between)
    return mask ? launch_sliced<true, true>(a, deep_rows, s)
                : launch_sliced<true, false>(a, deep_rows, s);
  return mask ? launch_sliced<false, true>(a, deep_rows, s)
              : launch_sliced<false, false>(a, deep_rows, s);
}

}  // namespace bsb
