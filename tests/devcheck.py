"""Device-side naive filters for the full-size parity tests (test
infrastructure): the reference checks scans against ``naive_filter`` over
the raw values (tests/helpers.py:35-52); at BASELINE sizes the same filter
runs on the GPU with torch and is packed into the reference word layout
(bitvector.py:3-5: bit i of word i // 32, LSB first)."""

import torch


def pack_bools(flags: torch.Tensor) -> torch.Tensor:
    """bool[n] (device) -> int32 words holding the uint32 bitvector words."""
    n = flags.numel()
    nw = -(-n // 32)
    out = torch.empty(nw, dtype=torch.int32, device=flags.device)
    sh = torch.arange(32, device=flags.device, dtype=torch.int32)
    step = 1 << 25  # words per chunk (bounded temporaries at 2^31+ rows)
    for w0 in range(0, nw, step):
        w1 = min(nw, w0 + step)
        f = torch.zeros((w1 - w0) * 32, dtype=torch.int32, device=flags.device)
        seg = flags[w0 * 32: min(n, w1 * 32)]
        f[: seg.numel()] = seg.to(torch.int32)
        out[w0:w1] = ((f.view(-1, 32) << sh).sum(1, dtype=torch.int64)).to(torch.int32)
    return out


def words_of(bv) -> torch.Tensor:
    """Device words of a DeviceBitVector."""
    return bv.dwords
