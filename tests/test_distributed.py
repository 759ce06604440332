"""Frame sharding and the counter all-reduce of the multi-GPU path, run with
the gloo backend, world size 2, on CPU.  Each rank decodes its own contiguous frame range
(with the CPU oracle standing in for the GPU decode in this host-logic test); the reduced
counters must equal a single-process run over all frames, for weak and strong sharding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1504_00353_b200.shard import allreduce_counters, frame_range, max_over_ranks, split_range
from seeded_inputs import bpsk_awgn_llr, draw, quantize_i8

N, K, EBN0, SEED = 256, 128, 1.5, 77


def _counts(first, count):
    mask = oracle.construct_ga(N, K, 2.0)
    bits, noise = draw(SEED, first, count, K, N)
    llr = quantize_i8(bpsk_awgn_llr(oracle.encode_systematic(mask, bits), noise, EBN0, K))
    dec = oracle.info_bits(mask, oracle.fastssc_decode(mask, llr))
    err = dec != bits
    return np.array([count, int(err.sum()), int(err.any(axis=1).sum())], np.int64)


def _worker(rank, world, port, mode, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = frame_range(rank, world, total // world) if mode == "weak" else split_range(rank, world, total)
    c = torch.from_numpy(_counts(first, count))
    allreduce_counters(c)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((c.tolist(), t))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode,total", [("weak", 96), ("strong", 101)])
def test_two_rank_counters_equal_single_process(mode, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, t = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = total if mode == "strong" else (total // 2) * 2
    want = _counts(0, frames).tolist()
    assert got == want
    assert t == 2.0  # MAX over ranks


def test_ranges():
    assert [frame_range(r, 4, 10) for r in range(4)] == [(0, 10), (10, 10), (20, 10), (30, 10)]
    parts = [split_range(r, 3, 10) for r in range(3)]
    assert parts == [(0, 4), (4, 3), (7, 3)]
    assert sum(c for _, c in parts) == 10
    with pytest.raises(ValueError):
        frame_range(4, 4, 10)
