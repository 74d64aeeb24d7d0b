"""Sampled parity at BASELINE.json's full sizes on 1 GPU, in the launch configuration bench.py times
(-m gpu): configs[1] (paper net 500:1500, batch 128) and the configs[4] network (512:2048 on
224x224x3, batch 256) unsplit.  See tests/full_size.py."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_paper_net_full_size_sampled(orc):
    from full_size import check_step, bench_setup
    dev = torch.device("cuda", 0)
    net, parts, pn, params, x, y = bench_setup(1, 0, None, dev)
    try:
        fails = check_step(pn, net, parts, params, x, y, 0, 1, lambda o: [o])
    finally:
        pn.close()
    assert not fails, "\n".join(fails)


def test_full_size_check_is_not_vacuous(orc):
    """Negative control: the same sampled check against an oracle given conv2 weights 0.5 % off
    (2.5x the TF32 tolerance) must flag the passes that read them, and only those."""
    from full_size import check_step, bench_setup
    dev = torch.device("cuda", 0)
    net, parts, pn, params, x, y = bench_setup(1, 0, None, dev)
    bad = dict(params)
    bad["w1"] = params["w1"] * 1.005
    try:
        fails = check_step(pn, net, parts, bad, x, y, 0, 1, lambda o: [o])
    finally:
        pn.close()
    text = "\n".join(fails)
    assert "conv2 forward" in text and "conv2 dgrad" in text, text
    assert "wgrad" not in text and "conv1 forward" not in text, text


def test_scaled_net_full_size_sampled(orc):
    import synth
    from full_size import bench_setup, check_step
    dev = torch.device("cuda", 0)
    net, parts, pn, params, x, y = bench_setup(1, 0, None, dev, net=synth.scaled_net(), B=256)
    try:
        fails = check_step(pn, net, parts, params, x, y, 0, 1, lambda o: [o], n=256)
    finally:
        pn.close()
        torch.cuda.empty_cache()
    assert not fails, "\n".join(fails)
