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
