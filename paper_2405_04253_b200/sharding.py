"""Data-parallel sharding of the FNT hot path across GPUs.

* CDC (config 4): one long stream per polarization is split into contiguous
  OUTPUT ranges, one per rank. out[n] = sum_k h[k] x[n + c - k] needs
  x[n + c - n_taps + 1 .. n + c]; the kernel works in whole 64-sample
  overlap-save blocks, so a rank that owns outputs [a, b) reads inputs from the
  start of block (a + c) // 32 minus one hop to the end of block (b - 1 + c) // 32
  (a halo of at most 63 samples each side, zeros outside [0, L)). No exchange is
  needed: halos are read from the input, and outputs do not overlap.
* AEQ / full chain (configs 3, 5): links are independent objects; each rank
  owns a contiguous range of links. A single stream cannot be split (the tap
  recursion is sequential, aeq.py:182-189).
* The only cross-rank traffic is reporting: timing maxima, sample counts, and
  (for sharded CDC streams) the exact integer decimation statistics, which are
  summed with an integer all-reduce so the decimation phase is identical to the
  unsharded decision.
"""

from __future__ import annotations

from dataclasses import dataclass

HOP = 32


@dataclass(frozen=True)
class RangeShard:
    rank: int
    out_first: int
    out_count: int
    x_first: int
    x_count: int


def balanced_split(total: int, parts: int, align: int = 1) -> list[tuple[int, int]]:
    """[start, count) per part, contiguous, sizes differing by at most `align`."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    units = -(-total // align) if align > 1 else total
    base, extra = divmod(units, parts)
    out, pos = [], 0
    for r in range(parts):
        n = (base + (1 if r < extra else 0)) * align
        n = max(0, min(n, total - pos))
        out.append((pos, n))
        pos += n
    return out


def input_window(out_first: int, out_count: int, length: int, n_taps: int) -> tuple[int, int]:
    """Inputs [x_first, x_first + x_count) the CDC kernel reads for an output range."""
    if out_count <= 0:
        return out_first, 0
    c = n_taps // 2
    b_lo = (out_first + c) // HOP
    b_hi = (out_first + out_count - 1 + c) // HOP
    lo = max(0, b_lo * HOP - HOP)
    hi = min(length, b_hi * HOP + HOP)
    return lo, max(0, hi - lo)


def cdc_range_shards(length: int, world: int, n_taps: int = 32, align: int = HOP) -> list[RangeShard]:
    shards = []
    for r, (a, n) in enumerate(balanced_split(length, world, align)):
        xf, xc = input_window(a, n, length, n_taps)
        shards.append(RangeShard(r, a, n, xf, xc))
    return shards


def link_shards(n_links: int, world: int) -> list[tuple[int, int]]:
    """[first_link, count) per rank for independent links (weak or strong scaling)."""
    return balanced_split(n_links, world)
