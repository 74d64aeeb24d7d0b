"""The SPMD host logic of the N>1 path on CPU: world_size-2 `gloo` process groups (-m "not gpu").

What a rank does outside the CUDA kernels is reproduced with torch.distributed on CPU:
  * probe times are all-gathered and every rank derives the SAME partition map with the C-ABI
    planner (cp_partition_plan is host-only) — checked by hashing the maps across ranks;
  * each rank evaluates the convolution of ITS OWN kernel slice (the oracle stands in for the
    GPU kernels here) and the channel all-gather in rank order reproduces the unsplit layer
    bitwise;
  * the all-reduce of per-rank partial dX equals the unsplit dgrad (north_star);
  * the wgrad of a rank's slice equals the rows of the unsplit wgrad, bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_1712_02546_b200 import build as b
        b.build()
        from paper_1712_02546_b200 import convpart as cp

        # 1) plan agreement from all-gathered "probe" times (rank-dependent, as on real devices)
        t = torch.tensor([1.0 + 0.4 * rank], dtype=torch.float64)
        times = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(times, t)
        times = [float(x.item()) for x in times]
        plan = cp.cp_partition_plan(times, 37)
        h = torch.tensor([hash(tuple(map(tuple, plan.as_tuple())))], dtype=torch.int64)
        hs = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(hs, h)
        assert all(int(x) == int(h) for x in hs), "ranks derived different partition maps"
        kb, kc, _ = plan.as_tuple()

        # 2) same input on every rank, own kernel slice, channel all-gather == unsplit (bitwise)
        x = synth.normal((3, 4, 12, 12), 1).astype(np.float64)
        w = synth.normal((37, 4, 5, 5), 2).astype(np.float64)
        bias = synth.normal((37,), 3).astype(np.float64)
        sl = slice(kb[rank], kb[rank] + kc[rank])
        mine = torch.from_numpy(oracle.conv_fwd(x, w[sl], bias[sl]))
        # uneven Eq. 1 slices: allgather-v as one broadcast per root (the library's grouped
        # ncclBroadcast path for unequal block widths)
        parts = []
        for r in range(world):
            buf = mine.clone() if r == rank else torch.zeros(3, kc[r], 8, 8, dtype=torch.float64)
            dist.broadcast(buf, src=r)
            parts.append(buf)
        full = torch.cat(parts, 1).numpy()
        assert np.array_equal(full, oracle.conv_fwd(x, w, bias))

        # 3) partial dX all-reduced == unsplit dX; wgrad rows local
        dy = synth.normal((3, 37, 8, 8), 4).astype(np.float64)
        part_dx = torch.from_numpy(oracle.conv_dgrad(dy, w, kb[rank], kb[rank] + kc[rank]))
        dist.all_reduce(part_dx)
        ref = oracle.conv_dgrad(dy, w)
        assert np.max(np.abs(part_dx.numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))
        dw_rows = oracle.conv_wgrad(dy[:, sl], x, 5, 5)
        assert np.array_equal(dw_rows, oracle.conv_wgrad(dy, x, 5, 5)[sl])
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")


def test_gloo_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
