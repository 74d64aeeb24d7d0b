"""conv2 wgrad error vs accumulation length at the scaled net (configs[4]) size: prints the sampled
max|gpu-ref|/max|ref| of every pass (tests/full_size.py) for the current CP_TC_SPLIT_WGRAD."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import full_size  # noqa: E402
import synth  # noqa: E402

full_size.TOL = {k: 0.0 for k in full_size.TOL}   # report every error
dev = torch.device("cuda", 0)
net, parts, pn, params, x, y = full_size.bench_setup(1, 0, None, dev, net=synth.scaled_net(), B=256)
fails = full_size.check_step(pn, net, parts, params, x, y, 0, 1, lambda o: [o], n=256)
print(f"CP_TC_SPLIT_WGRAD={os.environ.get('CP_TC_SPLIT_WGRAD', 'auto')}")
print("\n".join(f for f in fails if "wgrad" in f or "bias" in f))
