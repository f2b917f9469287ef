/*
 * bytestore_b200.h -- C ABI of the B200-native ByteStore scan/lookup hot path.
 *
 * This is the drop-in boundary under the reference's Python layout API
 * (reference: /root/reference/pkg/src/bytestore/, cited below as file:line).
 * The reference has no FFI of its own: its boundary is the Python surface
 * re-exported by __init__.py:10-52 and the string-keyed layout dispatch in
 * engine.py:172-221.  Each entry point below replaces one reference routine;
 * the ctypes binding a maintainer would add to the reference is shown in
 * INTEGRATION.md, and the package paper_2209_00220_b200 is that binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All array pointers are DEVICE pointers
 *    (cudaMalloc / torch allocations) unless the name says host.  `stream`
 *    is a cudaStream_t passed as void*; NULL means the legacy default stream.
 *  - Buffers are caller-allocated.  Functions never synchronise the stream
 *    except where documented ("syncs"): a value must come back to the host.
 *  - Bitvectors: uint32 words, bit i of row space = bit (i % 32) of word
 *    i / 32, LSB first (reference bitvector.py:1-6).  Words beyond
 *    ceil(n_rows/32) are never written; tail bits >= n_rows are written 0.
 *  - Status codes map to the reference's exceptions: BSB_EINVAL/BSB_ERANGE ->
 *    ValueError, BSB_ENOTFOUND -> LookupError, BSB_EKEY -> KeyError,
 *    BSB_ECUDA -> RuntimeError (CUDA error; bsb_last_error() has the text).
 */
#ifndef BYTESTORE_B200_H
#define BYTESTORE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSB_LANES 32          /* rows per block / bits per result word        */
#define BSB_TILE_BLOCKS 32    /* blocks per tile (one warp, lane = block)      */
#define BSB_TILE_ROWS 1024    /* rows per tile                                  */
#define BSB_MAX_LEVELS 8      /* slices per code (reference vbs.py:77-78)       */
#define BSB_MAX_CONJ 8        /* predicates per bsb_conj_scan call              */
#define BSB_STATS_WORDS 24    /* int64 counters written by the *_scan stats path */

enum bsb_status {
  BSB_OK = 0,
  BSB_EINVAL = 1,     /* bad argument / shape mismatch        -> ValueError   */
  BSB_ERANGE = 2,     /* value out of range (width, length)   -> ValueError   */
  BSB_ENOTFOUND = 3,  /* padded code not in dictionary        -> LookupError  */
  BSB_ECUDA = 4,      /* CUDA runtime error                   -> RuntimeError */
  BSB_EKEY = 5,       /* value missing from dictionary        -> KeyError     */
  BSB_EINDEX = 6      /* row id outside [0, n_rows)           -> IndexError   */
};

/* Operators: reference predicate.py:13-38 (Op). */
/* Bits of the device error word (err_dev) of the row-id lookups. */
#define BSB_ERR_NOTFOUND 1u
#define BSB_ERR_INDEX 2u

enum bsb_op { BSB_EQ = 0, BSB_NE = 1, BSB_LT = 2, BSB_LE = 3, BSB_GT = 4, BSB_GE = 5,
              BSB_BETWEEN = 6 };

/* Code-space predicate: reference predicate.py:62-95 (ResolvedPredicate).
 * trivial: -1 = real comparison, 0 = constant false, 1 = constant true.
 * length/length2 are BYTES (big-endian literal of that many bytes). */
typedef struct bsb_pred {
  int32_t op;
  int32_t trivial;
  uint64_t code;
  uint64_t code2;
  int32_t length;
  int32_t length2;
} bsb_pred;

/* Device-resident ByteSlice column (reference byteslice.py:34-49).
 * slices: n_slices planes of `stride` bytes each.  Inside every 32-row block
 * the 32 bytes of a plane are stored swizzled: row r of the block lives at
 * byte ((r & 7) << 2) | (r >> 3), so one
 * 256-bit load per lane gives SWAR-ready words.  stride is a multiple of
 * BSB_TILE_ROWS and >= n_rows; padding rows are zero. */
typedef struct bsb_byteslice {
  int64_t n_rows;
  int64_t stride;
  int32_t width_bits;
  int32_t n_slices;
  const uint8_t* slices;
} bsb_byteslice;

/* Device-resident PP-VBS column (reference vbs.py:42-65).
 * bs1:        first byte of every row, `stride` bytes, swizzled like ByteSlice.
 * exist[j]:   uint32 existence word per block of slice j+1 (vbs.py:101-104),
 *             `stride/32` words (row space, exactly the reference's M_{j+1}).
 * deep_mode selects how the deep slices (levels 2..max_len) are stored:
 *  BSB_DEEP_PACKED (0): deep[j] = slice j+1 packed in row order exactly like
 *             the reference (vbs.py:98-100); block_dir[j] = int64[stride/32+1]
 *             bytes of slice j+1 before block b (vbs.py:105-106).
 *  BSB_DEEP_SLICED (3): the deep rows form their own ByteSlice-like column:
 *             deep[j] (j = 1..max_len-1) holds byte j+1 of every deep row in
 *             32-deep-row "deep blocks", swizzled like bs1 (0-padded for rows
 *             without that byte); rexist[j] (j = 2..max_len-1) holds one uint32
 *             per deep block: bit i = deep row 32k+i has byte j+1.  Scanned with
 *             the ByteSlice SWAR compare, one lane per deep block.
 *             deep[0] (optional, SLICED only) holds byte 1 of every deep row
 *             in the same deep-block layout; with it (or with the
 *             deep1_shared zone map, which makes it unnecessary) scans run
 *             entirely in deep-row space for the deep rows.
 * deep allocations are padded by >= 64 bytes.  Index 0 of exist/block_dir/
 * rexist is unused (level 1 is bs1); index 0 of deep is unused except as
 * above. */
#define BSB_DEEP_PACKED 0
#define BSB_DEEP_SLICED 3 /* modes 1 and 2 (experimental round-1 layouts) were removed */
typedef struct bsb_vbs {
  int64_t n_rows;
  int64_t stride;
  int32_t max_len;
  int32_t deep_mode;
  const uint8_t* bs1;
  const uint8_t* deep[BSB_MAX_LEVELS];
  const uint32_t* exist[BSB_MAX_LEVELS];
  const int64_t* block_dir[BSB_MAX_LEVELS];
  int64_t deep_len[BSB_MAX_LEVELS];
  const uint32_t* rexist[BSB_MAX_LEVELS];
  /* Zone map of the deep rows' first byte (SLICED): 1 + the byte when every
   * deep row starts with the same byte, which lets scans settle level 1 of
   * the deep rows without reading deep[0]; 0 = not shared / unknown (the
   * zero-initialised default). */
  int32_t deep1_shared;
  int32_t reserved;
} bsb_vbs;

/* One column reference for bsb_conj_scan (engine.py:322-332). */
enum bsb_layout { BSB_LAYOUT_BYTESLICE = 0, BSB_LAYOUT_PPVBS = 1 };
typedef struct bsb_column_ref {
  int32_t layout;
  int32_t reserved;
  const bsb_byteslice* byteslice;  /* host pointers to the descriptors */
  const bsb_vbs* vbs;
} bsb_column_ref;

/* ----------------------------------------------------------------- misc */
const char* bsb_version(void);
/* Run-time tuning knobs (benchmarks and experiments; never change results;
 * a negative value restores the default): "ds_enable" (0 off, 1 on, 2
 * unmasked scans only), "ds_serial" (warp-cooperative pdep up to this many
 * blocks per tile), "ds_tiles" (tiles per super-tile, 0 = auto),
 * "ds_unroll" (0/1), "ds_zonemap" (0/1: settle level 1 from deep1_shared),
 * "sparse_ppm" (masked SLICED PP-VBS scans run the compacted kernel -- work
 * over the masked-in blocks only -- when the mask holds at most this many
 * rows per million, else scan the column whole and AND the mask into the
 * result words; the mask's row count is the chain's running count inside
 * bsb_conj_scan, a sampled estimate otherwise; default 60000, 0 = always the
 * latter), "ds_masked" (1: masked scans always scan whole), "dsm_cfg"
 * (compacted kernel shape 0..3), "conj_fuse" (0/1: fused ByteSlice pairs in
 * bsb_conj_scan), "stats_rows" (1: PP-VBS ScanStats through the
 * row-parallel kernel instead of the deep-row-space one), "ctas_per_sm"
 * (cap on the CTAs per SM of the persistent scan kernels, 0 = none: room for
 * a kernel of another stream; measured slower), "pair_bits" (row-bucket bits
 * of bsb_rows_bucket, 1..13), "dense_rows" (fused PP-VBS bitvector lookup:
 * selected rows per 1024-row tile from which deep-sector loads allocate in
 * L1; default 96), "coop_tiles" (fused bitvector lookups of columns of at
 * most this many 1024-row tiles run as ONE cooperative kernel -- per-warp
 * tile runs, totals exchanged across a grid barrier -- instead of tile
 * popcount + scan + lookup; default 2^14, 0 = never).  Unknown key:
 * BSB_EINVAL. */
int bsb_tune(const char* key, int64_t value);
const char* bsb_last_error(void);
/* Padded plane size for n rows (multiple of BSB_TILE_ROWS). */
int64_t bsb_stride_for(int64_t n_rows);

/* ------------------------------------------------------------ ByteSlice */
/* build_byteslice (byteslice.py:56-73): codes uint64[n_rows] -> swizzled,
 * left-aligned planes into slices[n_slices * stride] (caller-allocated,
 * n_slices = ceil(width_bits/8)).  Validates 1 <= width_bits <= 64 and
 * codes < 2^width (BSB_ERANGE; syncs to read the device check). */
int bsb_byteslice_build(const uint64_t* codes, int64_t n_rows, int32_t width_bits,
                        uint8_t* slices, int64_t stride, void* stream);
/* Same, from int64 ranks (Dictionary.encode_rows output, dictionary.py:381-397). */
int bsb_byteslice_build_ranks(const int64_t* ranks, int64_t n_rows, int32_t width_bits,
                              uint8_t* slices, int64_t stride, void* stream);
/* Reference (unswizzled) planes, uint8[n_slices][ceil(n/32)*32] -- parity helper. */
int bsb_byteslice_export(const bsb_byteslice* col, uint8_t* out, void* stream);

/* scan_byteslice (byteslice.py:109-140).  mask may be NULL (no input
 * bitvector).  out_words: ceil(n/32) words.  count: one uint64, overwritten;
 * NULL (without stats) = words only, like the reference's scan (no memset
 * node, no atomics).  Columns up to ~19M rows take a single-wave kernel
 * (every tile's sectors of a level in flight at once, launched with
 * programmatic stream serialization).
 * stats/depth may be NULL; when given, BETWEEN runs as two pipelined legs and
 * stats (BSB_STATS_WORDS int64, see bsb_stats_layout) / depth (int8 per
 * block) reproduce the reference ScanStats exactly (stats.py:18-84). */
int bsb_byteslice_scan(const bsb_byteslice* col, const bsb_pred* pred, const uint32_t* mask,
                       uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                       void* stream);

/* lookup_byteslice (byteslice.py:143-158) for a row-id list (any order,
 * duplicates allowed; output in input order).  Writes right-aligned codes to
 * out_codes (may be NULL) and, when rank_values (int64[dict size]) is given,
 * decoded values values[code] (dictionary.py:413-414) to out_values (int64,
 * may be NULL) and/or out_values32 (int32, may be NULL).  Without
 * rank_values, out_values32 receives the codes truncated to int32 (columns
 * whose codes are the values).  Row ids are checked against [0, n_rows)
 * inside the gather (an out-of-range id is never read; the reference raises
 * IndexError at the numpy fancy index, byteslice.py:154): with err_dev (a
 * caller-zeroed device word) the call does not synchronise and ORs
 * BSB_ERR_INDEX into *err_dev; with err_dev NULL it synchronises and returns
 * BSB_EINDEX. */
int bsb_byteslice_lookup_rows(const bsb_byteslice* col, const int64_t* rows, int64_t n_ids,
                              uint64_t* out_codes, const int64_t* rank_values,
                              int64_t* out_values, int32_t* out_values32, uint32_t* err_dev,
                              void* stream);

/* ----------------------------------------------------------------- PP-VBS */
/* build_vbs, pass 1 (vbs.py:68-82): validate lengths 1..8 and code widths,
 * return max_len and, per level j (1-based), the number of rows whose code
 * has a j-th byte: level_rows[j-1].  Syncs. */
int bsb_vbs_plan(const uint64_t* codes, const uint8_t* lens, int64_t n_rows,
                 int32_t* max_len_host, int64_t* level_rows_host, void* stream);
/* build_vbs, pass 2 (vbs.py:84-114): fills a descriptor whose arrays the
 * caller allocated from the plan (deep[j] >= level_rows[j] + 64 bytes). */
int bsb_vbs_build(const uint64_t* codes, const uint8_t* lens, const bsb_vbs* col,
                  void* stream);
/* Reference (unswizzled) first slice, uint8[ceil(n/32)*32] -- parity helper. */
int bsb_vbs_export_bs1(const bsb_vbs* col, uint8_t* out, void* stream);
/* Reference-packed slice `level` (2..max_len) into out_bytes (level_rows
 * bytes) and its reference block directory into out_dir (int64[nb+1]), for
 * either deep_mode -- parity helper. */
int bsb_vbs_export_level(const bsb_vbs* col, int32_t level, uint8_t* out_bytes,
                         int64_t* out_dir, void* stream);

/* scan_vbs (vbs.py:292-324): Alg. 3 with the existence shortcut.  Same
 * argument contract as bsb_byteslice_scan.  A literal longer than max_len
 * is BSB_ERANGE (the reference raises IndexError at vbs.py:274). */
int bsb_vbs_scan(const bsb_vbs* col, const bsb_pred* pred, const uint32_t* mask,
                 uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                 void* stream);

/* lookup_vbs (vbs.py:331-371) for a row-id list: padded codes
 * code << 8*(max_len - len) to out_padded (may be NULL); when sorted_padded
 * (uint64[n_dict], strictly increasing: ordered dictionaries, dictionary.py:
 * 370-373) and dict_values (int64[n_dict]) are given, also decode_padded
 * (dictionary.py:403-411) into out_values / out_values32 (either may be
 * NULL).  A code absent from the dictionary sets BSB_ENOTFOUND (syncs only
 * when decoding).  level_counts (uint64[BSB_MAX_LEVELS], may be NULL) is
 * overwritten with the number of looked-up rows owning a byte at each level
 * (LookupStats accounting, vbs.py:346-370).  err_dev as for
 * bsb_byteslice_lookup_rows (BSB_ERR_INDEX / BSB_ERR_NOTFOUND bits; NULL =
 * synchronise and return BSB_EINDEX / BSB_ENOTFOUND). */
int bsb_vbs_lookup_rows(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                        uint64_t* out_padded, const uint64_t* sorted_padded,
                        const int64_t* dict_values, int64_t n_dict, int64_t* out_values,
                        int32_t* out_values32, uint64_t* level_counts, uint32_t* err_dev,
                        void* stream);

/* Decode of looked-up codes to values (dictionary.py:403-414).
 *  kind 0: none (raw codes out)
 *  kind 1: rank table: value = values[code]            (decode_ranks)
 *  kind 2: sorted padded codes + values in that order   (decode_padded,
 *          binary search; any dictionary)
 *  kind 3: PPE tree (ppe_numerical dictionaries, dictionary.py:170-195):
 *          two dependent table reads + the value.  -1 = absent in every
 *          field; a node may be a code and a parent at once.
 *            e1[b1] (int64[256]) = child c (bits 0-31) | rank of the 1-byte
 *              code b1 (bits 32-63)
 *            e2[2*(c*256+b2)]   = rank of the 2-byte code (b1, b2)
 *            e2[2*(c*256+b2)+1] = leaf start | size << 32 | beta << 56: codes
 *              of length beta + 2 below (b1, b2), rank = start + suffix - 1,
 *              1 <= suffix <= size
 *          An absent code gives BSB_ENOTFOUND.  values = rank -> value. */
typedef struct bsb_decode {
  int32_t kind;
  int32_t reserved;
  const int64_t* values;
  const uint64_t* sorted_padded;
  int64_t n_dict;
  const int64_t* e1;
  const int64_t* e2;
} bsb_decode;

/* Fused bitvector-driven lookups (bitvector.py:71-72 + lookup_* + decode):
 * the set rows of `words` (n_rows = column rows) in ascending order, written
 * compactly to out_codes (uint64; ByteSlice right-aligned codes, PP-VBS padded
 * codes) and/or, with a decoder, out_values (int64) / out_values32 (int32).
 * No row-id array is materialised.  With n_out_dev given the call does not
 * synchronise: the number of rows written goes to that device scalar, or
 * UINT64_MAX when a code is not in the dictionary.  With n_out_dev NULL a
 * decoding call synchronises and returns BSB_ENOTFOUND for such a code. */
int bsb_byteslice_lookup_bits(const bsb_byteslice* col, const uint32_t* words,
                              const bsb_decode* dec, uint64_t* out_codes, int64_t* out_values,
                              int32_t* out_values32, uint64_t* n_out_dev, void* stream);
int bsb_vbs_lookup_bits(const bsb_vbs* col, const uint32_t* words, const bsb_decode* dec,
                        uint64_t* out_padded, int64_t* out_values, int32_t* out_values32,
                        uint64_t* n_out_dev, void* stream);
/* Row-id lookup of a PP-VBS column with a general decoder (kinds 0/2/3).
 * With err_dev (caller-zeroed device word) given the call does not
 * synchronise and ORs BSB_ERR_NOTFOUND into *err_dev for a code not in the
 * dictionary and BSB_ERR_INDEX for a row id outside [0, n_rows) (never
 * read); with err_dev NULL it synchronises and returns BSB_EINDEX /
 * BSB_ENOTFOUND. */
int bsb_vbs_lookup_rows_dec(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                            const bsb_decode* dec, uint64_t* out_padded, int64_t* out_values,
                            int32_t* out_values32, uint32_t* err_dev, void* stream);

/* ------------------------------------------------------- gather locality */
/* A row-id list for a gather (cfg3's unsorted ids): if rows[] (n_ids ids of
 * a column of n_rows rows) is not ascending, sorted_rows = the ids ordered by
 * row bucket (at most 2^16 buckets of consecutive rows; input order inside a
 * bucket) and perm[i] = the input position of sorted_rows[i]; a lookup of
 * sorted_rows walks the column in order and bsb_scatter puts its output back
 * in input order.  *was_sorted = 1 (outputs untouched) when the list looks
 * ascending (a sampled check of 4096 adjacent pairs: a mis-verdict only
 * skips the optimisation).  Syncs (the order check). */
int bsb_rows_sort(const int64_t* rows, int64_t n_ids, int64_t n_rows, int64_t* sorted_rows,
                  int64_t* perm, int32_t* was_sorted, void* stream);
/* The same locality without the sort or the perm array (lists of < 2^32 - 1
 * ids over columns of < 2^32 - 1 rows; BSB_EINVAL otherwise): pairs[i] =
 * row | position << 32, partitioned by row bucket (at most 2^13 buckets of
 * consecutive rows, at least 2^10 rows each; any order inside a bucket).  An
 * id outside [0, n_rows) becomes row 0xffffffff, which the pair lookups
 * report as BSB_ERR_INDEX like any other bad id.  Never synchronises.
 * unsorted_dev NULL: always partition.  Else *unsorted_dev (a device word) =
 * 0 when the list looks ascending (the sampled check of bsb_rows_sort) and
 * the partition kernels exit at once, 1 otherwise: the verdict stays on the
 * device and gates the pair lookups below. */
int bsb_rows_bucket(const int64_t* rows, int64_t n_ids, int64_t n_rows, uint64_t* pairs,
                    uint32_t* unsorted_dev, void* stream);
/* bsb_byteslice_lookup_rows / bsb_vbs_lookup_rows_dec over bsb_rows_bucket
 * pairs: out*[position] = the lookup of row, i.e. the row-id lookup of the
 * list the pairs were made from (byteslice.py:143-158 / vbs.py:331-371
 * applied to the given rows; output order = input order).  rows /
 * unsorted_dev NULL: the pairs are used.  With both given (the list and the
 * verdict bsb_rows_bucket left), *unsorted_dev == 0 gathers rows[] as given
 * instead -- the alternative that does not apply is launched and exits, so
 * the choice costs no host synchronisation. */
int bsb_byteslice_lookup_pairs(const bsb_byteslice* col, const uint64_t* pairs,
                               const int64_t* rows, const uint32_t* unsorted_dev, int64_t n_ids,
                               uint64_t* out_codes, const int64_t* rank_values,
                               int64_t* out_values, int32_t* out_values32, uint32_t* err_dev,
                               void* stream);
int bsb_vbs_lookup_pairs_dec(const bsb_vbs* col, const uint64_t* pairs, const int64_t* rows,
                             const uint32_t* unsorted_dev, int64_t n_ids, const bsb_decode* dec,
                             uint64_t* out_padded, int64_t* out_values, int32_t* out_values32,
                             uint32_t* err_dev, void* stream);
/* bsb_byteslice_lookup_rows / bsb_vbs_lookup_rows_dec with the locality
 * chosen from a sampled order check (4096 adjacent pairs): an ascending list
 * is gathered as given, any other through the bucket partition + pair gather.
 * Same arguments, same output.  On an idle, non-capturing stream the host
 * reads the verdict from a mapped word (a poll of ~10 us, no stream
 * synchronisation) and launches only the form that applies; otherwise both
 * forms are launched, each gated on the device-resident verdict (the one that
 * does not apply exits at once), so the call is graph-capturable and never
 * waits for work queued earlier.  Lists of fewer than 2 ids or sizes the
 * 32-bit pairs cannot hold are gathered as given. */
int bsb_byteslice_lookup_rows_auto(const bsb_byteslice* col, const int64_t* rows, int64_t n_ids,
                                   uint64_t* out_codes, const int64_t* rank_values,
                                   int64_t* out_values, int32_t* out_values32,
                                   uint32_t* err_dev, void* stream);
int bsb_vbs_lookup_rows_dec_auto(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                                 const bsb_decode* dec, uint64_t* out_padded,
                                 int64_t* out_values, int32_t* out_values32, uint32_t* err_dev,
                                 void* stream);
/* out[perm[i]] = in[i] for n elements of elem_bytes (4 or 8). */
int bsb_scatter(const void* in, const int64_t* perm, int64_t n, int32_t elem_bytes, void* out,
                void* stream);

/* ------------------------------------------------------------ bitvectors */
/* ResultBitVector.to_indices (bitvector.py:71-72): ascending int64 row ids of
 * the set bits into rows_out (capacity >= popcount); count written to
 * *n_out_host.  Syncs. */
int bsb_bits_to_rows(const uint32_t* words, int64_t n_rows, int64_t* rows_out,
                     int64_t* n_out_host, void* stream);
/* Same but with a row offset added (sharded global ids) and no sync: the
 * count is written to the device scalar n_out_dev. */
int bsb_bits_to_rows_async(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                           int64_t* rows_out, uint64_t* n_out_dev, void* stream);
/* Compaction of one row-range segment into a shared id array without a host
 * sync: ids row_offset + i of the set bits are written to
 * rows_out[*base_dev ...], base_dev a device int64 (e.g. the exclusive prefix
 * of the earlier segments' counts). */
int bsb_bits_to_rows_at(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                        const int64_t* base_dev, int64_t* rows_out, uint64_t* n_out_dev,
                        void* stream);
/* & | ~ and popcount (bitvector.py:84-125).  op: 0 = and, 1 = or, 2 = not
 * (b ignored), 3 = andnot (a & ~b).  Tail bits cleared. */
int bsb_bits_combine(int32_t op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                     int64_t n_rows, void* stream);
int bsb_bits_popcount(const uint32_t* words, int64_t n_rows, uint64_t* count, void* stream);

/* ------------------------------------------------------------ conjunction */
/* engine.execute's pipelined conjunction (engine.py:322-332) in one call:
 * predicate i sees the running result of predicates 0..i-1 as its input
 * mask (a chain of the per-layout scan kernels, no host sync); blocks already
 * zero load no slice bytes of later predicates.  Columns must share n_rows.
 * k <= BSB_MAX_CONJ. */
int bsb_conj_scan(int32_t k, const bsb_column_ref* cols, const bsb_pred* preds,
                  const uint32_t* mask, uint32_t* out_words, uint64_t* count, void* stream);

/* --------------------------------------------------------------- encoders */
/* build_frequency_table for numeric columns (dictionary.py:101-106) plus
 * encode_rows (dictionary.py:381-397) in one device sort:
 * values int64[n] -> distinct sorted values + counts (capacity n) and the
 * rank of every row.  *n_distinct_host receives the distinct count.  Syncs. */
int bsb_freq_table(const int64_t* values, int64_t n, int64_t* uniq_out, int64_t* counts_out,
                   int64_t* ranks_out, int64_t* n_distinct_host, void* stream);
/* Dictionary.encode_rows against an existing sorted table (binary search);
 * a value absent from the table -> BSB_EKEY (syncs). */
int bsb_encode_rows(const int64_t* values, int64_t n, const int64_t* table_values,
                    int64_t n_dict, int64_t* ranks_out, void* stream);
/* ppe_numerical (dictionary.py:148-196), HOST arrays: weights int64[n] ->
 * codes uint64[n], lengths uint8[n].  Stable top-255 tie-break. */
int bsb_ppe_numerical_host(const int64_t* weights_host, int64_t n, uint64_t* codes_host,
                           uint8_t* lengths_host);
/* Dictionary.row_codes (dictionary.py:399-401): gather per-row codes/lengths. */
int bsb_gather_codes(const int64_t* ranks, int64_t n, const uint64_t* dict_codes,
                     const uint8_t* dict_lens, uint64_t* codes_out, uint8_t* lens_out,
                     void* stream);
/* gen_zipf's inverse-CDF step (datagen.py:50-56): searchsorted(cdf, u,
 * side="right") for float64 uniforms u[n] over cdf[domain]. */
int bsb_zipf_from_uniform(const double* u, int64_t n, const double* cdf, int64_t domain,
                          int64_t* values_out, void* stream);

/* Layout of the stats buffer (int64):
 *   [0..7]   words_loaded per level     [8..15] bytes_loaded per level
 *   [16]     blocks_total               [17]    blocks_skipped
 *   [18]     levels (column K)          [19..23] reserved
 * mask_bytes is derived on the host: live_blocks * 4 * (min(len+1, K) - 1)
 * (vbs.py:286-287). */
void bsb_stats_layout(int32_t* words_off, int32_t* bytes_off, int32_t* total_off,
                      int32_t* skipped_off, int32_t* levels_off);

/* ------------------------------------------- baseline layouts (§8(f) row 4) */
/* Bit-Packed (bitpacked.py:1-150): code i in stream bits [i*w, (i+1)*w), most
 * significant bit first, bytes in stream order; stored as uint32 words whose
 * memory bytes ARE the reference stream (`bits`), zero padded to whole
 * 32-row groups plus two words.  w in 1..32. */
typedef struct bsb_bitpacked {
  int64_t n_rows;
  int32_t width_bits;
  int32_t reserved;
  const uint32_t* words;
} bsb_bitpacked;
/* words to allocate for n rows of width w (-1 on bad arguments) */
int64_t bsb_bitpacked_words_for(int64_t n_rows, int32_t width_bits);
/* build_bitpacked (bitpacked.py:36-52); a code >= 2^w -> BSB_ERANGE (syncs) */
int bsb_bitpacked_build(const int64_t* codes, int64_t n, int32_t width_bits, uint32_t* words,
                        void* stream);
/* scan_bitpacked (bitpacked.py:94-118): unpack + compare every code, input
 * mask post-AND-ed, no early stop, no ScanStats.  BETWEEN = code..code2. */
int bsb_bitpacked_scan(const bsb_bitpacked* col, const bsb_pred* pred, const uint32_t* mask,
                       uint32_t* out_words, uint64_t* count, void* stream);
/* lookup_bitpacked (bitpacked.py:127-143) of the set rows of `words`, in
 * ascending row order; decoder kind 0 (codes) or 1 (values[code]).  With
 * n_out_dev the row count lands there; out_* need capacity popcount. */
int bsb_bitpacked_lookup_bits(const bsb_bitpacked* col, const uint32_t* words,
                              const bsb_decode* dec, uint64_t* out_codes, int64_t* out_values,
                              int32_t* out_values32, uint64_t* n_out_dev, void* stream);

/* VBP / PE-VBP (vbp.py:1-212): plane j (0 = most significant) holds one
 * uint32 per 32-row block, planes[j * n_words + b]; kind PADDED stores
 * prefix-free codes zero-padded to w_max bits and aligns literals the same
 * way (code << (w_max - length), length in bits). */
#define BSB_VBP_PLAIN 0
#define BSB_VBP_PADDED 1
#define BSB_VBP_MAX_PLANES 32
#define BSB_VBP_STATS_WORDS 66
typedef struct bsb_vbp {
  int64_t n_rows;
  int32_t w_max;
  int32_t kind;
  const uint32_t* planes;
} bsb_vbp;
/* build_vbp (vbp.py:51-71): codes (already padded for PE-VBP) -> planes
 * (w_max * ceil(n/32) words); a code >= 2^w_max -> BSB_ERANGE (syncs). */
int bsb_vbp_build(const uint64_t* codes, int64_t n, int32_t w_max, uint32_t* planes,
                  void* stream);
/* scan_vbp (vbp.py:144-194): bit-serial, early stop per block; BETWEEN fused
 * (leg 2 sees leg 1's result as its mask).  stats (int64[BSB_VBP_STATS_WORDS],
 * may be NULL): [0..31] blocks loaded per plane (summed over legs; bytes =
 * 4 x), [64] blocks skipped by leg 1, [65] by leg 2; depth (int8 per block,
 * may be NULL) = max over legs -- the reference's merged ScanStats. */
int bsb_vbp_scan(const bsb_vbp* col, const bsb_pred* pred, const uint32_t* mask,
                 uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                 void* stream);
/* lookup_vbp (vbp.py:197-212) of the set rows of `words`, ascending row
 * order: padded codes, or values through decoder kind 1 (ranks) / 2 (sorted
 * padded codes, PE-VBP). */
int bsb_vbp_lookup_bits(const bsb_vbp* col, const uint32_t* words, const bsb_decode* dec,
                        uint64_t* out_codes, int64_t* out_values, int32_t* out_values32,
                        uint64_t* n_out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BYTESTORE_B200_H */
