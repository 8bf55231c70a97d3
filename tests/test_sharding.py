"""Multi-rank host logic on the CPU (gloo, world_size 2): range shards with the
overlap-save halo reproduce the unsharded CDC stream, link shards cover every
link once, and the exact integer decimation statistics all-reduce to the same
phase decision. The per-rank compute here is the CPU oracle (the test box has no
GPU); the GPU kernel's range interface is covered by
test_gpu_parity.py::test_cdc_bank_ranges_match_full_stream."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2405_04253_b200.sharding import (balanced_split, cdc_range_shards, input_window,
                                            link_shards)

TAP_RE = np.array([22, -4, -23, -6, 18, 20, 2, -17, -23, -16, -4, 8, 16, 21, 22, 23, 23, 23, 22,
                   21, 16, 8, -4, -16, -23, -17, 2, 20, 18, -6, -23, -4])
TAP_IM = np.array([6, 22, 0, -22, -13, 10, 23, 15, -2, -16, -22, -21, -16, -9, -4, -1, 0, -1, -4,
                   -9, -16, -21, -22, -16, -2, 15, 23, 10, -13, -22, 0, 22])


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_output(xr, xi, sh, L):
    """What rank sh.rank computes from ONLY its input window (oracle stands in for the kernel)."""
    wr = np.zeros(L, np.int64)
    wi = np.zeros(L, np.int64)
    wr[sh.x_first:sh.x_first + sh.x_count] = xr[sh.x_first:sh.x_first + sh.x_count]
    wi[sh.x_first:sh.x_first + sh.x_count] = xi[sh.x_first:sh.x_first + sh.x_count]
    yr, yi = O.cdc_direct(TAP_RE, TAP_IM, wr, wi)
    return yr[sh.out_first:sh.out_first + sh.out_count], yi[sh.out_first:sh.out_first + sh.out_count]


def _worker(rank, world, port, L, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    rng = np.random.default_rng(123)
    xr = rng.integers(-15, 16, L)
    xi = rng.integers(-15, 16, L)
    shards = cdc_range_shards(L, world, n_taps=32)
    sh = shards[rank]
    yr, yi = _shard_output(xr, xi, sh, L)
    # gather shard outputs (variable sizes -> pad to max)
    mx = max(s.out_count for s in shards)
    buf = torch.zeros((2, mx), dtype=torch.int64)
    buf[0, :sh.out_count] = torch.from_numpy(yr)
    buf[1, :sh.out_count] = torch.from_numpy(yi)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    # exact decimation statistics: integer sums per phase, all-reduced
    m2 = yr.astype(np.int64) ** 2 + yi.astype(np.int64) ** 2
    ph = (np.arange(sh.out_first, sh.out_first + sh.out_count) & 1)
    stats = torch.tensor([int(m2[ph == 0].sum()), int(m2[ph == 1].sum()),
                          int((m2[ph == 0] ** 2).sum()), int((m2[ph == 1] ** 2).sum())],
                         dtype=torch.int64)
    dist.all_reduce(stats, op=dist.ReduceOp.SUM)
    if rank == 0:
        full_r = np.concatenate([outs[r][0, :shards[r].out_count].numpy() for r in range(world)])
        full_i = np.concatenate([outs[r][1, :shards[r].out_count].numpy() for r in range(world)])
        ref_r, ref_i = O.cdc_direct(TAP_RE, TAP_IM, xr, xi)
        m2f = ref_r ** 2 + ref_i ** 2
        ph_f = np.arange(L) & 1
        exact = [int(m2f[ph_f == 0].sum()), int(m2f[ph_f == 1].sum()),
                 int((m2f[ph_f == 0] ** 2).sum()), int((m2f[ph_f == 1] ** 2).sum())]
        q.put((np.array_equal(full_r, ref_r) and np.array_equal(full_i, ref_i),
               stats.tolist() == exact))
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [20_011, 4096])
def test_gloo_world2_cdc_range_shards(L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, L, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok_out, ok_stats = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok_out, "sharded CDC differs from the unsharded stream"
    assert ok_stats, "all-reduced integer decimation statistics differ"


def test_halo_is_sufficient_for_every_split():
    rng = np.random.default_rng(7)
    L = 3000
    xr = rng.integers(-15, 16, L)
    xi = rng.integers(-15, 16, L)
    ref_r, ref_i = O.cdc_direct(TAP_RE, TAP_IM, xr, xi)
    for world in (1, 2, 3, 4, 8, 13):
        got_r = []
        for sh in cdc_range_shards(L, world):
            r, _ = _shard_output(xr, xi, sh, L)
            got_r.append(r)
        assert np.array_equal(np.concatenate(got_r), ref_r), world


def test_split_helpers():
    assert balanced_split(10, 3) == [(0, 4), (4, 3), (7, 3)]
    parts = balanced_split(1 << 31, 8, 32)
    assert sum(n for _, n in parts) == 1 << 31 and all(a % 32 == 0 for a, _ in parts)
    assert link_shards(4096, 8)[7] == (3584, 512)
    assert input_window(0, 32, 100, 32) == (0, 64)
    assert input_window(48, 32, 10_000, 32) == (32, 64)


def test_host_pipeline_segments_cover_exactly():
    """stream._segments (the pipelined host-buffer paths' input pieces / AEQ time
    segments): contiguous, aligned boundaries, exact cover, never empty pieces."""
    from paper_2405_04253_b200.stream import _segments
    for total in (0, 1, 63, 64, 65, 1000, 1 << 19, 12345):
        for parts in (1, 3, 4, 8, 100):
            for align in (1, 64):
                seg = _segments(total, parts, align)
                if total == 0:
                    assert seg == [(0, 0)]
                    continue
                assert seg[0][0] == 0 and seg[-1][1] == total
                assert all(a < b for a, b in seg)
                assert all(seg[i][1] == seg[i + 1][0] for i in range(len(seg) - 1))
                assert all(a % align == 0 for a, _ in seg)
                assert len(seg) <= parts
