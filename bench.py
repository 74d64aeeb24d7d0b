"""Benchmark: kernel-partitioned training of the paper's 500:1500 CIFAR-10-shaped CNN on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` (N>1 under torchrun, one rank
per GPU, NCCL).  Prints ONE JSON line on rank 0.

  * step   = one SGD training step of the whole network (conv1 fwd, AllGather, conv2 fwd,
             AllGather, FC + softmax loss head, FC bwd, conv2 dgrad + ReduceScatter of dX,
             conv2 wgrad, conv1 wgrad, SGD) — every conv layer kernel-partitioned across ranks
             (arXiv 1712.02546 §4, Alg. 1).
  * value  = images/s of the whole job: global batch / device-timed step time (max over ranks).
             Every rank processes the same B images (its own kernels), so the batch counts once.
  * e2e    = the same metric through the public API with host (pinned) buffers: the H2D copy of
             the step's images + labels and the D2H read of the loss are inside the timed region.
  * roofline = the dominant conv kernel (tcgen05 TF32 implicit GEMM), algorithmic FLOPs per launch
             / CUDA-event duration, against the TF32 peak derived from MEASURED_PEAKS.json.
  * cpu_baseline = the fp64 oracle (oracle/) timed on this host's cores on a bounded sample.
  * --impl reference = the oracle itself as the reference arm (this tier has no reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL_TF32_OVER_BF16 = 1.1 / 2.25  # B200_PROFILING.md nominal dense peaks (tf32 1.1, bf16 2.25 PF)



# the same metric string on both arms (the driver divides one by the other)
METRIC = "conv-layer train images/sec (whole-network SGD step, kernel-partitioned)"

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--net", default="500:1500")
    ap.add_argument("--math", default="tf32", choices=["tf32", "simt", "bf16"],
                    help="bf16 = NEXT row f4, report-only (bf16 operand copies; error outside the 2e-3 bar)")
    ap.add_argument("--probe-times", default=None,
                    help="comma-separated injected per-device probe times (s): Eq. 1 partition from these "
                         "instead of measuring (heterogeneous-device emulation, SURVEY §8(f) f3)")
    ap.add_argument("--partition", default="even", choices=["even", "probe"],
                    help="even split, or Eq. 1 from the paper's probe (times all-gathered)")
    ap.add_argument("--dx", default="rs", choices=["rs", "ar"])
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--head", default="partitioned", choices=["partitioned", "replicated"],
                    help="FC head: rank-local columns + AllReduce of logits, or all-gathered + replicated")
    ap.add_argument("--fused", default="on", choices=["on", "off"],
                    help="on: collectives fused into the GEMM epilogues over NVLink peer memory (channel "
                         "gather from the forward epilogue, dX reduce-scatter from the dgrad epilogue); "
                         "off: NCCL AllGather / ReduceScatter kernels")
    ap.add_argument("--lrn", action="store_true",
                    help="paper-literal net: Conv -> ReLU -> LRN -> Pool per conv layer (SPEC constants; NEXT row f2)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of a CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample duration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except Exception:
        pass
    if "bf16_tflops_sustained" in p:
        return {"tf32_sustained": p["bf16_tflops_sustained"] * NOMINAL_TF32_OVER_BF16,
                "tf32_burst": p["bf16_tflops"] * NOMINAL_TF32_OVER_BF16, "hbm": p.get("hbm_gbs", 6449.1),
                "source": "MEASURED_PEAKS.json bf16 x nominal tf32/bf16 (1.1/2.25)"}
    return {"tf32_sustained": 1400.0 * NOMINAL_TF32_OVER_BF16, "tf32_burst": 1590.0 * NOMINAL_TF32_OVER_BF16,
            "hbm": 6650.0, "source": "fallback B200_PROFILING.md x nominal tf32/bf16"}


NCU_FILES = ["r02_ncu_conv_tc.json", "r01_ncu_conv_tc.json"]   # newest first


def ncu_traffic(pass_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the conv2 kernel of this pass, from
    the newest committed ncu --set full summary (the longest launch of that pass = conv2)."""
    for fn in NCU_FILES:
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                rows = [r for r in json.load(f) if r.get("pass") == pass_name]
            if rows:
                return max(rows, key=lambda r: r.get("duration_us", 0))["traffic_bytes"], f"profiles/{fn}"
        except Exception:
            continue
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        self.t0 = time.time()
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def host_cores():
    """Cores this process may run on (the oracle's OpenMP team is sized to them)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_threads(n):
    """Size the oracle's OpenMP team: torchrun exports OMP_NUM_THREADS=1 to every rank, but the
    reference leg runs on rank 0 alone and may use the host's cores (libgomp is shared with the
    oracle's library)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
        return int(n)
    except OSError:
        return int(os.environ.get("OMP_NUM_THREADS", n))


def oracle_images_per_s(net, target_s, step=0):
    """Time the oracle's full training step on a bounded sample of the same workload."""
    import numpy as np

    import oracle
    import synth
    oracle.build()
    cores = oracle_threads(host_cores())
    params = {k: v.astype(np.float64) for k, v in synth.params(net, seed=42).items()}
    b, elapsed, done = 1, 0.0, 0
    while True:
        x, y = synth.images(b, 3, net.in_hw, net.in_hw, step=step)
        t0 = time.perf_counter()
        oracle.net_step(params, x.astype(np.float64), y, 0.01, net.layers())
        dt = time.perf_counter() - t0
        elapsed += dt
        done += b
        if elapsed >= target_s * 0.5 or dt * 2 > target_s:
            break
        b = max(1, min(64, int(b * max(2.0, (target_s - elapsed) / max(dt, 1e-3) * 0.5))))
    return done / elapsed, cores, f"{done} images of the B=128 step's workload ({net.name}), fp64 oracle net_step, {elapsed:.1f} s"


def run_reference(args):
    """The oracle as the reference arm: every step is the fp64 oracle's training step on a bounded
    sample of the B-image batch (b images, b calibrated once during the warm-up so that the whole run
    takes about --cpu-seconds); ms_per_step is the measured wall time of one such step."""
    import numpy as np

    import oracle
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    oracle.build()
    cores = oracle_threads(host_cores())
    net = synth.paper_net(args.net)
    params = {k: v.astype(np.float64) for k, v in synth.params(net, seed=42).items()}
    per_step_s = max(0.5, args.cpu_seconds / max(1, args.steps))
    b, times = 1, []
    for k in range(args.warmup + args.steps):
        x, y = synth.images(b, 3, net.in_hw, net.in_hw, step=k)
        t0 = time.perf_counter()
        oracle.net_step(params, x.astype(np.float64), y, 0.01, net.layers())
        dt = time.perf_counter() - t0
        if k < args.warmup:   # calibrate the sample size: about per_step_s of CPU work per step
            b = max(1, min(args.batch, int(round(b * per_step_s / max(dt, 1e-3)))))
        else:
            times.append(dt)
    dt = statistics.median(times)
    v = b / dt
    sample = (f"{b} of the B={args.batch} step's images per step ({net.name}), fp64 oracle net_step; median of "
              f"{len(times)} timed steps, {dt:.2f} s each")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "images_per_step": b,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"paper net {args.net}, CIFAR-10-shaped 32x32x3, batch "
                                                        f"{args.batch}, CPU fp64 oracle (bounded sample per step)",
                                            "global_batch": args.batch},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def _graph(step_fn, dev):
    """CUDA graph of one step (kernels + collectives + stream fork/join); returns (graph, launches)."""
    import torch

    from paper_1712_02546_b200 import convpart as cp
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    c0 = cp.cp_launch_count()
    with torch.cuda.graph(g):
        step_fn()
    n = cp.cp_launch_count() - c0
    g.replay()
    torch.cuda.synchronize(dev)
    return g, n


def _timed(run, steps, s, dev, flush, world, after=None):
    """Device time (ms) of `steps` calls of run(), each bracketed by CUDA events on `s`, L2 flushed
    between calls (outside the events); max over ranks of the total.  after(k) runs between steps."""
    import torch
    import torch.distributed as dist
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    for k in range(steps):
        if flush is not None:
            flush.fill_(k & 0xFF)
        ev[k][0].record(s)
        run()
        ev[k][1].record(s)
        torch.cuda.synchronize(dev)
        if after:
            after(k)
    total = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return total / steps


def _max_over_ranks(vals, dev, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return vals
    t = torch.tensor(vals, device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def _nccl_reference(parts, B, net, dev, world, steps=20):
    """NCCL AllGather / ReduceScatter of the step's A1 bytes over NVLink on their own (torch's NCCL
    process group, the same links): the collective-alone bandwidth the fused paths are compared with."""
    import torch
    import torch.distributed as dist
    Bp = (B + 31) // 32 * 32
    _, _, _, _, hp1 = net.shapes()[0]
    blk = hp1 * hp1 * Bp * max(parts[0].k_width[r] for r in range(world))   # floats per rank (equal blocks)
    src = torch.zeros(blk, device=dev)
    dst = torch.zeros(blk * world, device=dev)
    out = {}
    for name, fn in (("allgather", lambda: dist.all_gather_into_tensor(dst, src)),
                     ("reduce_scatter", lambda: dist.reduce_scatter_tensor(src, dst))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = _max_over_ranks([e0.elapsed_time(e1) / steps], dev, world)[0]
        moved = blk * 4 * (world - 1)      # bytes received (AG) / sent (RS) per rank
        out[name] = {"bytes_per_rank": moved, "ms": ms, "gbs_per_rank": moved / (ms / 1e3) / 1e9,
                     "frac_of_770": moved / (ms / 1e3) / 770e9}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_1712_02546_b200 import convpart as cp
    from paper_1712_02546_b200.net import PartitionedNet

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        sys.stdout.flush()
        fd = os.dup(1)
        os.dup2(2, 1)   # keep NCCL's init banner off stdout
        try:
            dist.init_process_group("nccl", device_id=dev)
        finally:
            sys.stdout.flush()
            os.dup2(fd, 1)
            os.close(fd)
    net = synth.scaled_net() if args.net == "scaled" else synth.paper_net(args.net)
    B = args.batch
    math = {"tf32": cp.CP_MATH_TF32, "simt": cp.CP_MATH_FP32_SIMT, "bf16": cp.CP_MATH_BF16}[args.math]
    align = 64 if math == cp.CP_MATH_BF16 else 8   # bf16: 64-element K-chunks need 64-slot widths

    # ---- communicator: unique id from rank 0 through torch.distributed (plumbing)
    comm = None
    if world > 1:
        uid = [cp.cp_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        # NCCL prints its version banner on stdout at init: keep stdout for the one JSON line
        sys.stdout.flush()
        saved_fd = os.dup(1)
        os.dup2(2, 1)
        try:
            comm = cp.cp_comm_create(uid[0], rank, world)
        finally:
            sys.stdout.flush()
            os.dup2(saved_fd, 1)
            os.close(saved_fd)

    # ---- partition map: even, or Eq. 1 from the paper's probe convolution (§4.1.1)
    probe_times = None
    if args.probe_times and world > 1:
        probe_times = [float(v) for v in args.probe_times.split(",")]
        if len(probe_times) != world:
            raise SystemExit(f"--probe-times needs {world} values")
        parts = [cp.cp_partition_plan(probe_times, K, align) for K in net.kernels]
    elif args.partition == "probe" and world > 1:
        d = cp.cp_conv_desc()
        c, h = net.shapes()[1][0], net.shapes()[1][1]
        d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = B, c, h, h, net.kernels[1], 5, 5
        d.bias, d.relu, d.pool, d.math, d.input_kind = 1, 1, 1, math, cp.CP_INPUT_GATHER
        d.in_part = cp.cp_partition_plan([1.0], c, align)
        d.out_part = cp.cp_partition_plan([1.0], net.kernels[1], align)
        d.rank, d.world = 0, 1
        scratch = torch.empty(cp.conv_part_probe_bytes(d), dtype=torch.uint8, device=dev)
        t = cp.conv_part_probe(d, scratch, warmups=1, reps=3)
        del scratch
        allt = [None] * world
        dist.all_gather_object(allt, t)
        probe_times = allt
        parts = [cp.cp_partition_plan(allt, K, align) for K in net.kernels]
    else:
        parts = [cp.cp_partition_plan([1.0] * world, K, align) for K in net.kernels]

    lrn = cp.LRN_DEFAULT if args.lrn else None
    pn = PartitionedNet(net.kernels, B, parts, rank=rank, comm=comm, math=math, device=dev, head=args.head,
                        in_hw=net.in_hw, fused=args.fused == "on", lrn=lrn)
    params = synth.params(net, seed=42)
    pn.load_params(params)
    x, y = synth.images(B, 3, net.in_hw, net.in_hw, step=0)
    x_host = torch.from_numpy(x).pin_memory()
    y_host = torch.from_numpy(y).pin_memory()
    pn.set_batch(x_host.to(dev), y_host.to(dev))
    s = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(dev)
    dx_mode = cp.CP_DX_REDUCE_SCATTER if args.dx == "rs" else cp.CP_DX_ALLREDUCE
    overlap = not args.no_overlap
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step_eager(head=True):
        # the current stream (torch's capture stream while a CUDA graph is being captured)
        pn.step(0.01, dx_mode, torch.cuda.current_stream(dev), cs, overlap, head=head)

    for _ in range(args.warmup):
        step_eager()
    torch.cuda.synchronize(dev)
    # live timing of conv2's three GEMM kernels inside the timed steps (external event records on the
    # launching stream, captured into the graph), and of the fused gather's push window (N > 1)
    cp.conv_part_timing(pn.layers[1], True)
    graph, launches_per_step = None, None
    if not args.no_graph:
        # CUDA graph of one whole step: removes the host launch path; every kernel in it is ours
        graph, launches_per_step = _graph(step_eager, dev)

    def step():
        if graph is not None:
            graph.replay()
        else:
            step_eager()
    if world > 1:
        dist.barrier()

    # ---- device-timed region: K steps, L2 flushed between steps (outside the step events)
    clocks = ClockSampler(local)
    clocks.start()
    live = {"fwd": [], "dgrad": [], "wgrad": [], "push": [], "rs": []}
    fused_gather = world > 1 and bool(pn.sym) and math == cp.CP_MATH_TF32
    # the library's fused-collective variants (environment, read per call; defaults: copy engines)
    gather_mode = "push" if os.environ.get("CP_GATHER_MODE") == "push" else "ce"
    rs_mode = os.environ.get("CP_RS_MODE") if os.environ.get("CP_RS_MODE") in ("push", "pull") else "ce"

    def read_live(k):
        # this step's kernel events, read before the next replay re-records them (device time only: the
        # host sync sits between steps, next to the L2 flush)
        for name, ps in (("fwd", 0), ("dgrad", 1), ("wgrad", 2)):
            live[name].append(cp.conv_part_kernel_time(pn.layers[1], ps))
        if fused_gather:
            for name, ps in (("push", 3), ("rs", 4)):
                try:
                    live[name].append(cp.conv_part_kernel_time(pn.layers[1], ps))
                except cp.ConvPartError:
                    pass
    # ---- the timed steps, device-timed (value) and end to end through the public API (e2e) interleaved
    # step by step, so both see the same clocks / power state (measured one loop after the other, the
    # later loop ran on a hotter, more power-capped GPU: scripts/e2e_probe.py).
    # e2e: pinned host images/labels in, loss out to the host, per step.  Input pipeline: step k+1's
    # images/labels travel host -> device on a copy stream (pinned source, two staging buffers) while
    # step k computes, inside step k's timed window (its end waits for them); step 0's copy is issued
    # inside its own window.
    # Each e2e step starts with a device copy staging -> the network's input buffer and ends with the
    # loss read back to pinned host memory, which the host then reads.  L2 flushed before every step.
    h2d = x_host.numel() * x_host.element_size() + y_host.numel() * y_host.element_size()
    d2h = 4
    loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
    cpy = torch.cuda.Stream(dev)
    stage = [(torch.empty_like(pn.x), torch.empty_like(pn.labels)) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def prefetch(k):
        j = k & 1
        with torch.cuda.stream(cpy):
            cpy.wait_event(free[j])
            stage[j][0].copy_(x_host.reshape(-1), non_blocking=True)
            stage[j][1].copy_(y_host, non_blocking=True)
            ready[j].record(cpy)
    for j in range(2):
        free[j].record(s)
    e2e_graphs = None
    if graph is not None:
        # the e2e step as one graph per staging buffer, the network reading its images / labels straight
        # from that buffer (no device copies ahead of the step: as graph memcpy nodes they cost ~20 us of
        # copy-engine latency per step), so the host enqueues one launch per step
        def e2e_body(j):
            prev = pn.bind_input(stage[j][0], stage[j][1])
            try:
                step_eager()
            finally:
                pn.bind_input(*prev)
        e2e_graphs = [_graph(lambda j=j: e2e_body(j), dev)[0] for j in range(2)]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    host_losses = []
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    n0 = cp.cp_launch_count()
    for k in range(args.steps):
        # device-timed step
        if flush is not None:
            flush.fill_(k & 0xFF)
        ev[k][0].record(s)
        step()
        ev[k][1].record(s)
        torch.cuda.synchronize(dev)
        read_live(k)
        # end-to-end step
        j = k & 1
        if flush is not None:
            flush.fill_(k & 0xFF)
        e2e_ev[k][0].record(s)
        if k == 0:
            cpy.wait_stream(s)   # step 0's copy starts inside its own window
            prefetch(0)
        s.wait_event(ready[j])
        # the step is enqueued before the next input's copy, so the host's enqueue work does not sit
        # between the window's start and the step (the L2 flush ahead of it covers the launch)
        if e2e_graphs is not None:
            e2e_graphs[j].replay()   # the step on staging buffer j, one graph launch
        else:
            pn.x.copy_(stage[j][0])
            pn.labels.copy_(stage[j][1])
            step()
        free[j].record(s)
        if k + 1 < args.steps:
            # step k+1's inputs travel host -> device while step k computes (other staging buffer, free
            # since step k-1's graph ended); the window closes only after they landed
            prefetch(k + 1)
        loss_host.copy_(pn.head["loss"][:1], non_blocking=True)
        if k + 1 < args.steps:
            s.wait_event(ready[(k + 1) & 1])
        e2e_ev[k][1].record(s)
        e2e_ev[k][1].synchronize()
        host_losses.append(float(loss_host[0]))
    torch.cuda.synchronize(dev)
    launches = (cp.cp_launch_count() - n0) // 2 if graph is None else launches_per_step * args.steps
    ms_per_step = _max_over_ranks([sum(a.elapsed_time(b) for a, b in ev) / args.steps], dev, world)[0]
    value = B / (ms_per_step / 1e3)
    # the timed window is tens of ms; keep the same load (identical, untimed steps) until the
    # sampler has seen >= 1.5 s so the clock record is meaningful (step count from the max-over-ranks
    # ms_per_step: identical on every rank, the steps hold collectives)
    for _ in range(min(2000, int(1500.0 / max(ms_per_step, 0.05)) + 1)):
        step()
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    clk["window"] = "timed steps + e2e steps + identical untimed steps to >= 1.5 s"
    e2e_ms = _max_over_ranks([sum(a.elapsed_time(b) for a, b in e2e_ev) / args.steps], dev, world)[0]
    e2e_value = B / (e2e_ms / 1e3)
    loss = pn.loss()

    # ---- per-pass kernel timing of conv2 (the dominant kernels) on a no-collective clone
    L2d = pn.descs[1]
    h2 = cp.conv_part_create(L2d, None)
    b2 = pn.buf[1]
    ws2 = torch.empty_like(b2["ws"])
    y2 = b2["y"].clone()
    sv2 = b2["saved"].clone()
    dw2 = torch.empty_like(b2["dw"])
    db2 = torch.empty_like(b2["db"])
    dx2 = torch.empty_like(b2["dx"])
    a1 = pn.buf[0]["y"]
    da2 = pn.head["da"]
    tim = {"fwd": [], "wgrad": [], "dgrad": []}
    for r in range(6):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if flush is not None:
            flush.fill_(r)
        e[0].record(s)
        cp.conv_part_forward(h2, a1, b2["w"], b2["b"], y2, sv2, ws2, s, s)
        e[1].record(s)
        cp.conv_part_backward_filter(h2, da2, sv2, y2, a1, dw2, db2, ws2, s)
        e[2].record(s)
        cp.conv_part_backward_data(h2, da2, sv2, y2, b2["w"], dx2, cp.CP_DX_LOCAL, ws2, s, s)
        e[3].record(s)
        torch.cuda.synchronize(dev)
        if r:
            tim["fwd"].append(e[0].elapsed_time(e[1]))
            tim["wgrad"].append(e[1].elapsed_time(e[2]))
            tim["dgrad"].append(e[2].elapsed_time(e[3]))
    cp.conv_part_destroy(h2)
    del ws2, y2, sv2, dw2, db2, dx2

    # ---- conv stage: the same step with the head replaced by the fixed dA2 it produced
    g_conv, _ = (_graph(lambda: step_eager(head=False), dev) if graph is not None else (None, None))
    conv_ms = _timed((lambda: g_conv.replay()) if g_conv is not None else (lambda: step_eager(head=False)),
                     args.steps, s, dev, flush, world)
    del g_conv

    # ---- N > 1: the same ranks' compute with no cross-rank exchange, the 1-GPU step on this box, and
    # NCCL's collectives alone on the same bytes (context for the NVLink fraction)
    compute_ms, one_gpu, nccl_ref = None, None, None
    if world > 1:
        pc = PartitionedNet(net.kernels, B, parts, rank=rank, comm=None, math=math, device=dev, head=args.head,
                            in_hw=net.in_hw, fused=False, lrn=lrn)
        pc.load_params(params)
        pc.set_batch(x_host.to(dev), y_host.to(dev))
        run_c = lambda: pc.step(0.01, cp.CP_DX_LOCAL, torch.cuda.current_stream(dev), cs, overlap)  # noqa: E731
        for _ in range(2):
            run_c()
        gc, _ = _graph(run_c, dev) if graph is not None else (None, None)
        compute_ms = _timed((lambda: gc.replay()) if gc is not None else run_c, args.steps, s, dev, flush, world)
        del gc
        pc.close()
        del pc
        torch.cuda.empty_cache()
        nccl_ref = _nccl_reference(parts, B, net, dev, world)
        if rank == 0:
            p1 = [cp.cp_partition_plan([1.0], K, align) for K in net.kernels]
            po = PartitionedNet(net.kernels, B, p1, rank=0, comm=None, math=math, device=dev, in_hw=net.in_hw, lrn=lrn)
            po.load_params(params)
            po.set_batch(x_host.to(dev), y_host.to(dev))
            run_o = lambda: po.step(0.01, dx_mode, torch.cuda.current_stream(dev), cs, overlap)  # noqa: E731
            for _ in range(args.warmup):
                run_o()
            go, _ = _graph(run_o, dev) if graph is not None else (None, None)
            one_ms = _timed((lambda: go.replay()) if go is not None else run_o, args.steps, s, dev, flush, 1)
            del go
            po.close()
            del po
            torch.cuda.empty_cache()
            one_gpu = {"value": B / (one_ms / 1e3), "ms_per_step": one_ms}
        dist.barrier()

    Kr2 = parts[1].k_count[rank]
    C2, H2o = net.kernels[0], net.shapes()[1][3]
    flop_pass = 2.0 * B * Kr2 * C2 * 25 * H2o * H2o   # algorithmic MACs x2 of one conv2 pass, own slice
    pk = peaks()
    per = {k: statistics.median(v) for k, v in tim.items()}
    # roofline: the dominant conv2 GEMM kernel, its average launch duration measured live in the
    # timed steps (max over ranks: the slowest rank sets the step)
    live_ms = dict(zip(("fwd", "dgrad", "wgrad"), _max_over_ranks(
        [statistics.fmean(live[k]) for k in ("fwd", "dgrad", "wgrad")], dev, world)))
    push_ms = rs_ms = None
    if fused_gather:
        push_ms, rs_ms = _max_over_ranks([statistics.fmean(live[k]) if live[k] else -1.0 for k in ("push", "rs")],
                                         dev, world)
    dom = max(live_ms, key=live_ms.get)
    achieved = flop_pass / (live_ms[dom] / 1e3) / 1e12

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, cores, sample = oracle_images_per_s(net, args.cpu_seconds)
            cpu = {"value": v, "unit": "images/s", "cores": cores, "kind": "oracle", "sample": sample}
        # algorithmic training FLOPs per image (11.368 GFLOP for the paper net):
        # conv1 fwd + wgrad, conv2 fwd + dgrad + wgrad, 2 FLOP per MAC (head: negligible)
        (c1, _, k1, o1, hp1), (c2, _, k2, o2, hp2) = net.shapes()
        per_img = 2.0 * (2 * k1 * c1 * 25 * o1 * o1 + 3 * k2 * c2 * 25 * o2 * o2)
        step_flop = per_img * B
        # ONE peak per line: burst for a timed window of tens of ms, the sustained figure (MEASURED_PEAKS'
        # 4 s back-to-back run) once the timed steps themselves last a second or more (scaled net); the
        # contraction's own dtype: TF32 = measured bf16 x nominal tf32/bf16, BF16 = measured bf16
        window_s = args.steps * ms_per_step / 1e3
        sustained = window_s >= 1.0
        bf16 = math == cp.CP_MATH_BF16
        scale = 1.0 / NOMINAL_TF32_OVER_BF16 if bf16 else 1.0
        peak = (pk["tf32_sustained"] if sustained else pk["tf32_burst"]) * scale
        other = (pk["tf32_burst"] if sustained else pk["tf32_sustained"]) * scale
        kind = "kind::f16 (bf16 operands)" if bf16 else "kind::tf32"
        peak_note = (f" ({'sustained' if sustained else 'burst'}: the timed window is {window_s * 1e3:.0f} ms; "
                     f"{'burst' if sustained else 'sustained'} = {other:.0f})")
        if bf16:
            peak_note = " (bf16: MEASURED_PEAKS.json bf16 as measured)" + peak_note
        traffic, traffic_src = ncu_traffic(dom) if world == 1 else (None, None)
        line = {
            "metric": METRIC,
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {cp.CP_MATH_TF32: "tf32", cp.CP_MATH_BF16: "bf16"}.get(math, "f32"), "data": "synthetic",
            "config": {
                "workload": f"{net.name} (conv5x5 {net.kernels[0]} -> {'LRN -> ' if args.lrn else ''}pool -> conv5x5 "
                            f"{net.kernels[1]} -> {'LRN -> ' if args.lrn else ''}pool -> FC {net.fc_in}->10 -> softmax), "
                            f"{net.in_hw}x{net.in_hw}x3 synthetic images, batch {B}",
                "global_batch": B, "partition": [list(p.k_count[:p.n_ranks]) for p in parts],
                "partition_source": ("Eq.1 from injected times" if args.probe_times else "Eq.1 from probe")
                                    if probe_times else "even",
                "probe_times_s": probe_times, "dx_collective": args.dx, "overlap_wgrad_with_dx_reduce": overlap,
                "head": pn.head_mode, "cuda_graph": graph is not None,
                "lrn": dict(cp.LRN_DEFAULT) if args.lrn else None,
                "collectives": (f"NVLink peer memory, no NCCL kernels: gather = {gather_mode} (ce: copy engines "
                                "copy the own block into every peer's copy on the comm stream while conv2 forward "
                                "computes its own block first, arrival flags; push: the forward kernel's warp 3 "
                                f"pushes it), dX reduce-scatter = {rs_mode} (ce: owners fetch their block's partials "
                                "with the copy engines while wgrad runs; push: dgrad epilogue peer stores), "
                                "rank-order sum" if pn.sym else "NCCL AllGather / ReduceScatter")
                               if world > 1 else "none (N=1)",
                "parallelism": f"kernel-split x{world}",
                "l2": "flushed between timed steps (256 MiB write outside the step events)" if flush is not None
                      else "not flushed (step working set > 126 MB L2)"},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms,
                    "note": "pinned H2D of the step's images + labels (prefetched on a copy stream inside the previous "
                            "step's window), one graph launch per step holding the D2D copies into the net's input and "
                            "the step, D2H of the loss and its host read every step"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": f"conv2 {dom} (tcgen05 {kind} implicit GEMM)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": f"{traffic_src} (ncu --set full, same kernel, P=1)" if traffic_src else None,
                         "flop_per_launch": flop_pass, "launch_ms": live_ms[dom],
                         "launch_ms_source": "CUDA events around the GEMM launch inside the timed graph "
                                             "replays (conv_part_timing), mean over the timed steps, max over ranks",
                         "kernel_ms_live": live_ms,
                         "peak_source": (pk["source"] if not bf16 else "MEASURED_PEAKS.json bf16") + peak_note,
                         "conv2_pass_ms_alone": per,
                         "conv2_pass_tflops_alone": {k: flop_pass / (v / 1e3) / 1e12 for k, v in per.items()}},
            # whole-step algorithmic FLOP rate over the same peak as roofline.frac, times the N GPUs
            "tc_frac_whole_step": step_flop / (ms_per_step / 1e3) / 1e12 / (peak * world),
            "conv_stage": {"value": B / (conv_ms / 1e3), "unit": "images/s", "ms_per_step": conv_ms,
                           "what": "the same step with the FC/softmax head replaced by the fixed dA2 it produced "
                                   "(conv layers, their gathers and dX sums, wgrad, SGD of the conv slices)"},
            "clocks": clk, "loss": loss, "loss_host_last": host_losses[-1] if host_losses else None,
        }
        if world > 1:
            Bp = (B + 31) // 32 * 32
            blk1 = [hp1 * hp1 * Bp * parts[0].k_width[r] * 4 for r in range(world)]
            blk2 = [hp2 * hp2 * Bp * parts[1].k_width[r] * 4 for r in range(world)]
            others1 = sum(blk1) - blk1[rank]
            egress = blk1[rank] * (world - 1) + others1           # gather push + dX partials to the owners
            if pn.head_mode == "replicated":
                egress += blk2[rank] * (world - 1)
            push_bytes = blk1[rank] * (world - 1)
            exposed = ms_per_step - compute_ms
            line["speedup_vs_1"] = ({"value": value / one_gpu["value"], "one_gpu_value": one_gpu["value"],
                                     "one_gpu_ms_per_step": one_gpu["ms_per_step"],
                                     "measured": "same box, rank 0's GPU, same config at N=1, CUDA graph"}
                                    if one_gpu else None)
            line["breakdown_ms"] = {
                "step": ms_per_step,
                "compute_only": compute_ms,
                "exposed_comm": exposed,
                "head": ms_per_step - conv_ms,
                "conv_stage": conv_ms,
                "conv2_gemms_live": sum(live_ms.values()),
                "note": "compute_only = the same ranks' kernels with no cross-rank exchange (comm=None, LOCAL dX, "
                        "each rank's slice; CUDA graph); exposed_comm = step - compute_only; head = step - conv_stage "
                        "(FC fwd/bwd, softmax, logits AllReduce); cf. the paper's Comm/Conv/Comp split, Fig. 8 "
                        "(P:L408-412)"}
            line["nvlink"] = {
                "link_peak_gbs": 770.0,
                "link_peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                "egress_bytes_per_rank": egress,
                "gather": {"mode": gather_mode, "bytes_pushed": push_bytes,
                           "window_ms": push_ms if push_ms and push_ms > 0 else None,
                           "gbs": push_bytes / (push_ms / 1e3) / 1e9 if push_ms and push_ms > 0 else None,
                           "frac_of_770": push_bytes / (push_ms / 1e3) / 770e9 if push_ms and push_ms > 0 else None,
                           "how": ("CUDA events on the comm stream around the copy-engine copies of the own block "
                                   "into every peer's copy (+ one flag per peer), mean over timed steps, max over "
                                   "ranks; overlapped with the conv2 forward's own-block MMAs" if gather_mode == "ce"
                                   else "globaltimer window inside the conv2 forward kernel: first chunk claimed -> "
                                   "last chunk's arrival released (warp 3 of every running CTA), mean over timed "
                                   "steps, max over ranks; overlapped with the forward's own-block MMAs")},
                "reduce_scatter": ({"mode": "ce", "bytes_received": push_bytes,
                                    "window_ms": rs_ms if rs_ms and rs_ms > 0 else None,
                                    "gbs": push_bytes / (rs_ms / 1e3) / 1e9 if rs_ms and rs_ms > 0 else None,
                                    "frac_of_770": push_bytes / (rs_ms / 1e3) / 770e9 if rs_ms and rs_ms > 0 else None,
                                    "how": "CUDA events on the comm stream around the owner's copy-engine fetch of "
                                           "its block's partials from every peer (after all ready flags), mean over "
                                           "timed steps, max over ranks; overlapped with conv2 wgrad"}
                                   if rs_mode == "ce" else
                                   {"mode": rs_mode, "bytes_sent": others1, "window_ms": live_ms["dgrad"],
                                    "gbs_lower_bound": others1 / (live_ms["dgrad"] / 1e3) / 1e9,
                                    "how": "dgrad epilogue peer stores spread over the whole dgrad kernel (push) or "
                                           "SM loads by the owner (pull): bytes / dgrad time is a lower bound"}),
                "exposed_comm_ms": exposed,
                "step_avg_egress_frac_of_770": egress / (ms_per_step / 1e3) / 770e9,
                "nccl_alone": nccl_ref}
        if bf16:
            line["report_only"] = ("NEXT row f4: bf16 GEMM operands (kind::f16), fp32 accumulate; parity ~1e-2 "
                                   "of max|ref|, outside the north_star 2e-3 bar - not the headline mode")
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    # teardown: the graph holds work of our communicator -> free it first, sync, then the comm
    torch.cuda.synchronize(dev)
    if graph is not None:
        del graph
        e2e_graphs = None
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    pn.close()
    if comm is not None:
        cp.cp_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
