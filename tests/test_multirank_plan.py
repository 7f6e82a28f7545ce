"""Multi-GPU host logic on CPU: sharding, the global comb plan and the census
rebalance, exercised by world-size 2/3 gloo process groups.

Every rank runs the same C-ABI plan functions the CUDA driver runs
(hwwg_shard_range / hwwg_comb_plan / hwwg_rebalance_plan); particles move with
torch.distributed send/recv in place of the driver's NCCL send/recv. The
rebalanced next-step source must equal a single global comb of the
rank-ordered concatenated census (popctrl.cpp:7-42) — exactly, since the test
weights are integers and every fp64 sum is exact."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2512_19925_b200 as hw
from paper_2512_19925_b200 import hww


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def global_comb(weights, target, frac):
    """popctrl.cpp:15-37 on one bank: index of the particle each tooth copies."""
    W = float(np.sum(weights))
    spacing = W / target
    offset = frac * spacing
    cum = np.cumsum(weights)
    out = []
    i = 0
    for k in range(target):
        T = offset + k * spacing
        while i < len(cum) and not (T < cum[i]):
            i += 1
        out.append(i if i < len(cum) else len(cum) - 1)
    return np.array(out), spacing


def local_teeth(weights, origin, spacing, offset, k_lo, k_hi):
    """The device teeth kernel (k_comb_teeth_range): first local particle with
    T_k < origin + prefix."""
    prefix = np.cumsum(weights)
    idx = []
    for k in range(k_lo, k_hi):
        T = offset + k * spacing
        j = int(np.searchsorted(origin + prefix, T, side="right"))
        idx.append(min(j, len(prefix) - 1))
    return np.array(idx, dtype=np.int64)


def test_shard_ranges_partition():
    for H in (1, 7, 1000, 10**6 + 3):
        for world in (1, 2, 3, 8):
            spans = [hww.shard_range(H, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            for a, b in zip(spans, spans[1:]):
                assert a[1] == b[0]


def test_comb_plan_partitions_teeth():
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 8):
        w = rng.integers(0, 50, world).astype(float)
        w[0] += 1.0
        target = 97
        frac = 0.37
        ranges = [hww.comb_plan(w, r, target, frac) for r in range(world)]
        assert ranges[0][3] == 0 and ranges[-1][4] == target
        for a, b in zip(ranges, ranges[1:]):
            assert a[4] == b[3]
        # same answer as the single global comb on a bank of one particle per rank
        idx, _ = global_comb(w, target, frac)
        for r, (sp, off, org, lo, hi) in enumerate(ranges):
            assert np.all(idx[lo:hi] == r) or hi == lo


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)
        n_local = [5, 40, 17][rank]
        w_local = rng.integers(1, 9, n_local).astype(np.float64)  # integer: exact sums
        gid = np.arange(n_local) + 1000 * rank  # particle identity
        wt = torch.tensor([w_local.sum()], dtype=torch.float64)
        allw = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allw, wt)
        rank_w = np.array([float(x) for x in allw])
        target, frac = 53, 0.61
        plans = [hww.comb_plan(rank_w, q, target, frac) for q in range(world)]
        sp, off, org, k_lo, k_hi = plans[rank]
        teeth = gid[local_teeth(w_local, org, sp, off, k_lo, k_hi)] if k_hi > k_lo else \
            np.zeros(0, np.int64)
        klo = [p[3] for p in plans]
        khi = [p[4] for p in plans]
        send, first, recv = hww.rebalance_plan(klo, khi, rank, target)
        lo, hi = hww.shard_range(target, rank, world)
        mine = np.full(hi - lo, -1, np.int64)
        reqs = []
        for q in range(world):
            if send[q]:
                sl = teeth[int(first[q]) - k_lo: int(first[q]) - k_lo + int(send[q])]
                if q == rank:
                    mine[int(first[q]) - lo: int(first[q]) - lo + int(send[q])] = sl
                else:
                    reqs.append(dist.isend(torch.from_numpy(sl.copy()), dst=q))
        for q in range(world):
            if recv[q] and q != rank:
                buf = torch.zeros(int(recv[q]), dtype=torch.int64)
                dist.recv(buf, src=q)
                d0 = max(klo[q], lo) - lo
                mine[d0: d0 + int(recv[q])] = buf.numpy()
        for r in reqs:
            r.wait()
        # send/recv consistency: what q sends to me == what I expect from q
        allsend = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allsend, torch.from_numpy(send.astype(np.int64)))
        for q in range(world):
            assert int(allsend[q][rank]) == int(recv[q])
        # gather shards and the banks; rank 0 compares with one global comb
        size = torch.tensor([hi - lo])
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, size)
        mx = int(max(s.item() for s in sizes))
        pad = torch.full((mx,), -2, dtype=torch.int64)
        pad[: hi - lo] = torch.from_numpy(mine)
        shards = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(shards, pad)
        nmax = 64
        wl = torch.zeros(nmax, dtype=torch.float64)
        wl[:n_local] = torch.from_numpy(w_local)
        banks = [torch.zeros(nmax, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(banks, wl)
        ns = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ns, torch.tensor([n_local]))
        if rank == 0:
            new_src = np.concatenate([shards[q][: int(sizes[q])].numpy() for q in range(world)])
            all_w = np.concatenate([banks[q][: int(ns[q])].numpy() for q in range(world)])
            all_id = np.concatenate([np.arange(int(ns[q])) + 1000 * q for q in range(world)])
            ref_idx, _ = global_comb(all_w, target, frac)
            result_q.put((new_src.tolist(), all_id[ref_idx].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_comb_rebalance_matches_global_comb(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want
