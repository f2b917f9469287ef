"""Multi-rank sharded scan on CPU: world_size=2 over gloo.

The per-shard scan is the oracle (this box has no GPU); the sharding plan,
the single count all_gather, offsets, global row ids and dictionary merge are
the product's code (paper_2209_00220_b200.sharded).  Result: concatenated
shard bitvectors, summed counts and gathered row ids equal the unsharded run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2209_00220_b200 import sharded as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N_TOTAL = 70_000 + 123


def _column():
    return O.gen_zipf(1.1, 16, N_TOTAL, 500)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vals = _column()
        r0, r1 = S.shard_range(N_TOTAL, world, rank)
        local = vals[r0:r1]
        lu, lc = np.unique(local, return_counts=True)
        gu, gc = S.merge_frequency_tables(torch.from_numpy(lu), torch.from_numpy(lc))
        gu, gc = gu.numpy(), gc.numpy()
        d = O.OracleDict(gu, gc, "prefix_preserving")
        col = O.vbs_build(*d.row_codes(d.encode_rows(local)))
        srt = np.sort(vals)
        lo, hi = int(srt[int(0.8 * N_TOTAL)]), int(srt[int(0.95 * N_TOTAL)])
        pred = d.encode_literal("BETWEEN", lo, hi)

        def local_scan(a, b):
            assert (a, b) == (r0, r1)
            w, _ = O.vbs_scan(col, pred)
            return w, torch.tensor([O.words_count(w)], dtype=torch.int64)

        res = S.sharded_scan(local_scan, N_TOTAL)
        ids = S.global_row_ids(res)
        all_ids = S.gather_row_ids(res, ids)
        flags = O.words_to_bools(res.local_bits, r1 - r0)
        tot = S.global_sum(torch.tensor([int(local[flags].sum())]))
        words = torch.from_numpy(res.local_bits.view(np.int32).copy())
        sizes = [None] * world
        dist.all_gather_object(sizes, (res.r0, res.r1, words.numpy().tolist()))
        q.put((rank, res.global_count, res.offset, res.counts, all_ids.numpy().tolist(),
               sizes, gu.tolist() == np.unique(vals).tolist(), int(tot.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scan_matches_unsharded(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    vals = _column()
    d = O.OracleDict.from_values(vals, "prefix_preserving")
    col = O.vbs_build(*d.row_codes(d.encode_rows(vals)))
    srt = np.sort(vals)
    lo, hi = int(srt[int(0.8 * N_TOTAL)]), int(srt[int(0.95 * N_TOTAL)])
    want, _ = O.vbs_scan(col, d.encode_literal("BETWEEN", lo, hi))
    want_rows = O.words_to_rows(want, N_TOTAL)
    shards = out[0][5]
    words = np.concatenate([np.array(w, np.int32).view(np.uint32) for _, _, w in shards])
    assert np.array_equal(words, want)                 # bit-exact concatenation
    off = 0
    for rank, total, offset, counts, ids, _, dict_ok, vsum in out:
        assert dict_ok                                 # merged dictionary == global table
        assert vsum == int(vals[want_rows].sum())      # SUM: local sums + one all_reduce
        assert total == len(want_rows) == sum(counts)
        assert offset == off
        off += counts[rank]
        assert ids == want_rows.tolist()               # gathered ascending global ids


def test_shard_range_alignment():
    for n in (1, 1023, 1024, 5000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [S.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and (a0 % 1024 == 0 or a0 == n)


# ---------------------------------------------------------------- cfg5 plan
# The bench's cfg5 table (bench_cfg5.Cfg5Table) on CPU: 8 fixed segments
# owned in contiguous runs (sharded.owned_segments), exact global quantiles of
# uint32 codes by the radix select over all ranks (global_nearest_rank_u32),
# global per-value counts by one all_reduce, per-segment oracle scans, and the
# AND's global row ids at each rank's exclusive-prefix offset.

SEG = 4096
NSEG = 8


def _seg_values(ci, s):
    import bench_cfg5 as C
    if ci < 2:
        return C.gen_host(ci, "uniform", s, SEG).astype(np.int64)
    return O.gen_zipf(1.1, 12, SEG, C.chunk_seed(ci, s))


def _cfg5_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        segs = list(S.owned_segments(NSEG, world, rank))
        raw = {ci: [_seg_values(ci, s) for s in segs] for ci in range(4)}
        n_total = NSEG * SEG
        qs = [S.global_nearest_rank_u32([torch.from_numpy(v + (1 << 31)) for v in raw[ci]],
                                        [x], n_total)[0] for ci, x in ((0, 0.10), (1, 0.50))]
        dicts = []
        for ci in (2, 3):
            w = torch.zeros(1 << 12, dtype=torch.int64)
            for v in raw[ci]:
                w += torch.bincount(torch.from_numpy(v), minlength=1 << 12)
            dist.all_reduce(w)
            u = torch.nonzero(w).flatten()
            dicts.append(O.OracleDict(u.numpy(), w[u].numpy(), "prefix_preserving"))
        z0lo = int(np.sort(np.concatenate([_seg_values(2, s) for s in range(NSEG)]))[
            int(0.8 * n_total)]) if rank == 0 else 0
        t = torch.tensor([z0lo])
        dist.broadcast(t, 0)
        z0lo = int(t.item())
        local_ids, local_cnt = [], 0
        for si, s in enumerate(segs):
            run = None
            for ci in range(4):
                v = raw[ci][si]
                if ci < 2:
                    planes = O.bs_build((v + (1 << 31)).astype(np.uint64), 32)
                    p = O.pred_compare("LT" if ci == 0 else "GE", qs[ci], 4)
                    run, _ = O.bs_scan(planes, 32, SEG, p, run)
                else:
                    d = dicts[ci - 2]
                    col = O.vbs_build(*d.row_codes(d.encode_rows(v)))
                    p = (d.encode_literal("GE", z0lo) if ci == 2 else
                         d.encode_literal("LE", 40))
                    run, _ = O.vbs_scan(col, p, run)
            rows = O.words_to_rows(run, SEG) + s * SEG
            local_ids.extend(rows.tolist())
            local_cnt += len(rows)
        counts, total, offset = S.exchange_counts(torch.tensor([local_cnt], dtype=torch.int64))
        q.put((rank, segs, qs, total, offset, counts, local_ids))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_cfg5_segment_plan_matches_one_rank(world):
    """Sharding the cfg5 table over 2 / 4 ranks (gloo) gives the 1-rank
    quantiles, dictionaries and AND row ids, each rank's ids at its
    exclusive-prefix offset of the global id array."""
    results = {}
    for w in (1, world):
        port = _free_port()
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_cfg5_worker, args=(r, w, port, q)) for r in range(w)]
        for p in procs:
            p.start()
        out = sorted(q.get(timeout=300) for _ in procs)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        results[w] = out
    one = results[1][0]
    all_ids = one[6]
    assert len(all_ids) == one[3] > 0
    segs_seen = []
    for rank, segs, qs, total, offset, counts, ids in results[world]:
        assert qs == one[2]                      # global quantiles identical at every world
        assert total == one[3]
        assert ids == all_ids[offset:offset + len(ids)]
        segs_seen += segs
    assert segs_seen == list(range(NSEG))
