"""Multi-GPU parity of the kernel-partitioned step over real NCCL collectives (torchrun, one rank
per GPU).  Launched by tests/test_gpu_multi.py; exits non-zero on any mismatch.

Checks (north_star invariants):
  * every rank holds the same gathered conv outputs (AllGather along channels), bitwise;
  * the gathered outputs equal the oracle's unsplit layer on the same inputs (TF32 tolerance);
  * summed partial dX (ReduceScatter / AllReduce) equals the oracle's unsplit dgrad;
  * each rank's dW / db slice equals the oracle's rows (decision replay);
  * the replicated head (loss, FC update) is bitwise identical on all ranks;
  * the paper net (BASELINE configs[2], and configs[3]'s batch 1024 with an Eq. 1 partition) and
    the scaled net (configs[4]) at full size, sampled outputs of every pass.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import TOL, rel_err, unpack  # noqa: E402
from paper_1712_02546_b200 import convpart as cp  # noqa: E402
from paper_1712_02546_b200.net import PartitionedNet  # noqa: E402


def _log(rank, msg):
    """progress on stderr (rank 0): locates a failing case in the torchrun log"""
    if rank == 0:
        print(f"[multi_gpu_check] {msg}", file=sys.stderr, flush=True)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    uid = [cp.cp_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = cp.cp_comm_create(uid[0], rank, world)
    failures = []
    uneven = [1.0 + 0.35 * r for r in range(world)]
    for mode_name, dx_mode, times, head, fused in [
            ("even+RS", cp.CP_DX_REDUCE_SCATTER, [1.0] * world, "replicated", False),
            ("eq1+AR", cp.CP_DX_ALLREDUCE, uneven, "replicated", False),
            ("even+RS+partitioned-head", cp.CP_DX_REDUCE_SCATTER, [1.0] * world, "partitioned", False),
            ("eq1+RS+partitioned-head", cp.CP_DX_REDUCE_SCATTER, uneven, "partitioned", False),
            # f1: gather fused into the forward epilogue, dX reduce-scatter fused into the dgrad epilogue
            # (peer stores over NVLink + arrival flags), even / uneven (Eq. 1) / skewed partitions
            ("even+RS+fused", cp.CP_DX_REDUCE_SCATTER, [1.0] * world, "replicated", True),
            ("eq1+RS+fused+partitioned-head", cp.CP_DX_REDUCE_SCATTER, uneven, "partitioned", True),
            ("skewed+RS+fused+partitioned-head", cp.CP_DX_REDUCE_SCATTER, [1.0] + [12.0] * (world - 1),
             "partitioned", True),
            ("eq1+AR+fused-gather+partitioned-head", cp.CP_DX_ALLREDUCE, uneven, "partitioned", True),
            # ranks with zero kernels in a layer: the last rank owns no conv1 kernel (an empty
            # input block of conv2: empty push, zero partial), rank 0 no conv2 kernel (copy-engine gather)
            ("zero-kernel-ranks+RS+fused+partitioned-head", cp.CP_DX_REDUCE_SCATTER, "zero", "partitioned", True),
            ("zero-kernel-ranks+RS+fused+replicated-head", cp.CP_DX_REDUCE_SCATTER, "zero", "replicated", True)]:
        _log(rank, mode_name)
        net = synth.NetSpec(kernels=(36, 72), in_hw=20, name="multi")
        B = 40
        if times == "zero":
            c1 = [36 // (world - 1)] * (world - 1)
            c1[0] += 36 - sum(c1)
            c2 = [0] + [72 // (world - 1)] * (world - 1)
            c2[1] += 72 - sum(c2)
            parts = [cp.cp_partition.from_counts(c1 + [0]), cp.cp_partition.from_counts(c2)]
        else:
            parts = [cp.cp_partition_plan(times, K) for K in net.kernels]
        params = synth.params(net, seed=21, std=0.05, bias_std=0.01)
        x, y = synth.images(B, 3, 20, 20, step=3)
        pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, device=dev, in_hw=20, head=head,
                            fused=fused)
        pn.load_params(params)
        pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
        s = torch.cuda.current_stream(dev)
        cs = torch.cuda.Stream(dev)
        pn.forward(s, cs)
        torch.cuda.synchronize(dev)
        hp = [8, 2]
        rep = []
        for i, K in enumerate(net.kernels):
            if head == "partitioned" and i == len(net.kernels) - 1:
                # rank-local last layer: assemble the full map from every rank's own block
                a_own = unpack(pn.buf[i]["y"], B, K, hp[i], parts[i])
                k0, kr = parts[i].k_begin[rank], parts[i].k_count[rank]
                pieces = [None] * world
                dist.all_gather_object(pieces, a_own[:, k0:k0 + kr])
                a = np.concatenate(pieces, 1)
            else:
                a = unpack(pn.buf[i]["y"], B, K, hp[i], parts[i])
                allv = [None] * world
                dist.all_gather_object(allv, a.tobytes())
                if any(v != allv[0] for v in allv):
                    failures.append(f"{mode_name}: gathered output of conv{i + 1} differs across ranks")
            kr = parts[i].k_count[rank]
            am = torch.zeros(max(B * kr * hp[i] * hp[i], 1), dtype=torch.uint8, device=dev)
            if kr:
                cp.cp_unpack_saved(pn.buf[i]["saved"], B, hp[i], hp[i], parts[i], rank, am)
            mine = am[: B * kr * hp[i] * hp[i]].reshape(B, kr, hp[i], hp[i]).cpu().numpy()
            codes = [None] * world
            dist.all_gather_object(codes, mine)
            rep.append({"a": a, "argmax": np.concatenate([c for c in codes if c.shape[1]], 1)})
        p64 = {k: v.astype(np.float64) for k, v in params.items()}
        tr = oracle.net_step(p64, x.astype(np.float64), y, 0.01, net.layers(), replay=rep)
        # forward parity per layer on identical inputs (GPU's own previous output as input)
        z1 = oracle.conv_fwd(x.astype(np.float64), p64["w0"], p64["b0"])
        a1, _ = oracle.relu_pool_fwd(z1)
        e = rel_err(rep[0]["a"], a1)
        if e > TOL[cp.CP_MATH_TF32]:
            failures.append(f"{mode_name}: conv1 fwd rel err {e:.2e}")
        z2 = oracle.conv_fwd(rep[0]["a"], p64["w1"], p64["b1"])
        a2, _ = oracle.relu_pool_fwd(z2)
        e = rel_err(rep[1]["a"], a2)
        if e > TOL[cp.CP_MATH_TF32]:
            failures.append(f"{mode_name}: conv2 fwd rel err {e:.2e}")
        pn.backward(dx_mode, s, cs, overlap=True)
        torch.cuda.synchronize(dev)
        # summed partial dX of conv2 = gradient w.r.t. A1 (this rank's block for RS, all for AR)
        dy2 = oracle.unpool_relu_bwd(tr["da1"], rep[1]["argmax"], rep[1]["a"])
        ref_da1 = oracle.conv_dgrad(dy2, p64["w1"])
        got = unpack(pn.buf[1]["dx"], B, net.kernels[0], 8, parts[0])
        k0, kr = parts[0].k_begin[rank], parts[0].k_count[rank]
        sl = slice(k0, k0 + kr) if dx_mode == cp.CP_DX_REDUCE_SCATTER else slice(0, net.kernels[0])
        if kr or dx_mode != cp.CP_DX_REDUCE_SCATTER:
            e = rel_err(got[:, sl], ref_da1[:, sl])
            if e > TOL[cp.CP_MATH_TF32]:
                failures.append(f"{mode_name}: summed dX rel err {e:.2e}")
        loss = pn.loss()
        losses = [None] * world
        dist.all_gather_object(losses, loss)
        if any(v != losses[0] for v in losses):
            failures.append(f"{mode_name}: loss differs across ranks {losses}")
        if abs(loss - tr["loss"]) > TOL[cp.CP_MATH_TF32] * abs(tr["loss"]):
            failures.append(f"{mode_name}: loss {loss} vs oracle {tr['loss']}")
        # weight gradients of this rank's slices (oracle with the GPU's own replayed decisions)
        pn.sgd(0.01, s)
        torch.cuda.synchronize(dev)
        new = pn.export_params()
        for i in range(2):
            kb, kr = parts[i].k_begin[rank], parts[i].k_count[rank]
            if not kr:
                continue
            upd = new[f"w{i}"] - params[f"w{i}"][kb:kb + kr]
            ref = tr["new_params"][f"w{i}"][kb:kb + kr] - p64[f"w{i}"][kb:kb + kr]
            e = rel_err(upd, ref)
            if e > 5e-3:
                failures.append(f"{mode_name}: conv{i + 1} weight update rel err {e:.2e}")
        if head == "replicated":
            fc = [None] * world
            dist.all_gather_object(fc, new["wfc"].tobytes())
            if any(v != fc[0] for v in fc):
                failures.append(f"{mode_name}: replicated FC weights differ across ranks")
            fc_ref = tr["new_params"]["wfc"] - p64["wfc"]
            fc_got = new["wfc"] - params["wfc"]
        else:
            k0, kr = parts[1].k_begin[rank], parts[1].k_count[rank]
            cols = lambda m: m.reshape(m.shape[0], -1, 4)[:, k0:k0 + kr].reshape(m.shape[0], -1)  # noqa: E731
            fc_ref = cols(tr["new_params"]["wfc"] - p64["wfc"])
            fc_got = new["wfc"] - cols(params["wfc"])
        if fc_got.size:
            e = rel_err(fc_got, fc_ref)
            if e > 5e-3:
                failures.append(f"{mode_name}: FC weight update rel err {e:.2e}")
        pn.close()

    # Paper-literal net (Conv -> ReLU -> LRN -> Pool, NEXT row f2) over real collectives: every rank
    # holds the pooled maps and codes of all channels, so the oracle replays them directly.
    for fused in (False, True):
        net = synth.NetSpec(kernels=(36, 72), in_hw=20, name="multi-lrn")
        B = 40
        lrn = {"depth": 5, "alpha": 0.05, "beta": 0.75, "bias": 2.0}
        parts = [cp.cp_partition_plan(uneven, K) for K in net.kernels]
        params = synth.params(net, seed=23, std=0.05, bias_std=0.01)
        x, y = synth.images(B, 3, 20, 20, step=4)
        pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, device=dev, in_hw=20, fused=fused, lrn=lrn)
        pn.load_params(params)
        pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
        s = torch.cuda.current_stream(dev)
        cs = torch.cuda.Stream(dev)
        pn.forward(s, cs)
        torch.cuda.synchronize(dev)
        rep = []
        for i, K in enumerate(net.kernels):
            ho = pn.buf[i]["hw"]
            rep.append({"a": unpack(pn.buf[i]["yp"], B, K, ho // 2, parts[i]),
                        "argmax": np.rint(unpack(pn.buf[i]["codes"].float(), B, K, ho // 2, parts[i])).astype(np.uint8),
                        "pre": unpack(pn.buf[i]["y"], B, K, ho, parts[i])})
        pn.backward(cp.CP_DX_REDUCE_SCATTER, s, cs, overlap=True)
        pn.sgd(0.01, s)
        torch.cuda.synchronize(dev)
        new = pn.export_params()
        p64 = {k: v.astype(np.float64) for k, v in params.items()}
        layers = [dict(L, lrn=lrn) for L in net.layers()]
        tr = oracle.net_step(p64, x.astype(np.float64), y, 0.01, layers, replay=rep)
        name = f"lrn{'+fused' if fused else ''}"
        if abs(pn.loss() - tr["loss"]) > TOL[cp.CP_MATH_TF32] * abs(tr["loss"]):
            failures.append(f"{name}: loss {pn.loss()} vs oracle {tr['loss']}")
        for i in range(2):
            kb, kr = parts[i].k_begin[rank], parts[i].k_count[rank]
            if kr:
                e = rel_err(new[f"w{i}"] - params[f"w{i}"][kb:kb + kr],
                            tr["new_params"][f"w{i}"][kb:kb + kr] - p64[f"w{i}"][kb:kb + kr])
                if e > 5e-3:
                    failures.append(f"{name}: conv{i + 1} weight update rel err {e:.2e}")
        e = rel_err(new["wfc"] - params["wfc"], tr["new_params"]["wfc"] - p64["wfc"])
        if e > 5e-3:
            failures.append(f"{name}: FC weight update rel err {e:.2e}")
        pn.close()

    # Several back-to-back steps (eager, then CUDA-graph replays) with the fused collectives vs NCCL:
    # exercises the arrival-flag resets and the overwrite guards across steps (a missed flag or an
    # early overwrite shows up as a diverging loss).
    net = synth.NetSpec(kernels=(36, 72), in_hw=20, name="multi")
    B = 40
    parts = [cp.cp_partition_plan([1.0] * world, K) for K in net.kernels]
    params = synth.params(net, seed=22, std=0.05, bias_std=0.01)
    s = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(dev)
    curves = {}
    for fused in (False, True):
        pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, device=dev, in_hw=20, head="partitioned",
                            fused=fused)
        pn.load_params(params)
        seq, graph = [], None
        for it in range(8):
            x, y = synth.images(B, 3, 20, 20, step=10 + it)
            pn.set_batch(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
            if it < 4:
                pn.step(0.05, cp.CP_DX_REDUCE_SCATTER, s, cs, True)
            else:
                if graph is None:
                    torch.cuda.synchronize(dev)
                    graph = torch.cuda.CUDAGraph()
                    cap = torch.cuda.Stream(dev)
                    cap.wait_stream(s)
                    with torch.cuda.graph(graph, stream=cap):
                        pn.step(0.05, cp.CP_DX_REDUCE_SCATTER, cap, cs, True)
                    s.wait_stream(cap)
                    # the capture did not execute: run the step that was just captured
                graph.replay()
            torch.cuda.synchronize(dev)
            seq.append(pn.loss())
        del graph
        torch.cuda.synchronize(dev)
        pn.close()
        curves[fused] = seq
    a, b = np.array(curves[False]), np.array(curves[True])
    if not np.all(np.abs(a - b) <= 2e-3 * np.abs(a)):
        failures.append(f"fused vs NCCL collectives over 8 steps: losses {b.tolist()} vs {a.tolist()}")

    # BASELINE configs[2] / configs[4] at full size in bench.py's launch configuration (even partition,
    # fused collectives), sampled parity per pass (tests/full_size.py)
    from full_size import bench_setup, check_step

    def allgather(o):
        out = [None] * world
        dist.all_gather_object(out, o)
        return out

    for name, head, net, B, times in [
            ("paper net", "partitioned", None, 128, None), ("paper net", "replicated", None, 128, None),
            ("paper net B=1024, Eq. 1 partition (configs[3])", "partitioned", None, 1024, uneven),
            ("scaled net (configs[4])", "partitioned", synth.scaled_net(), 256, None)]:
        _log(rank, f"full size: {name}, {head} head")
        net, parts, pn, params, x, y = bench_setup(world, rank, comm, dev, net=net, B=B, head=head, times=times)
        failures += [f"{name}, {head} head: {m}" for m in check_step(pn, net, parts, params, x, y, rank, world,
                                                                     allgather, n=256)]
        pn.close()
        torch.cuda.empty_cache()
    cp.cp_comm_destroy(comm)
    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.destroy_process_group()
    if rank == 0:
        flat = [f"rank {r}: {m}" for r, fl in enumerate(allf) for m in fl]
        print("\n".join(flat) if flat else f"multi-GPU parity OK on {world} ranks")
        sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
