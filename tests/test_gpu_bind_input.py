"""bench.py's end-to-end input path (-m gpu): PartitionedNet.bind_input makes the step read its images /
labels straight from the buffers a host -> device copy filled (one CUDA graph per staging buffer),
instead of copying them into the network's own input first (set_batch).

* the same batch through bind_input and through set_batch gives bitwise the same loss and parameters
  (the kernels read the same values; only the pointer differs);
* a graph captured while a staging buffer is bound follows that buffer's contents: refilling it with
  another batch and replaying gives the loss an eager step on that batch gives (the graph holds the
  staging pointer, not a copy);
* bind_input returns the previous pair and rejects buffers of the wrong size / dtype.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1712_02546_b200 import convpart as cp


def _net():
    from paper_1712_02546_b200.net import PartitionedNet, plan_even
    net = synth.NetSpec(kernels=(24, 40), in_hw=20, name="small")
    pn = PartitionedNet(net.kernels, 40, plan_even(net.kernels, 1), math=cp.CP_MATH_TF32, in_hw=20)
    pn.load_params(synth.params(net, seed=21, std=0.05, bias_std=0.01))
    return pn


def _params(pn):
    return [t.detach().clone() for b in pn.buf for t in (b["w"], b["b"])] + \
        [pn.head["wfc"].detach().clone(), pn.head["bfc"].detach().clone()]


def test_bind_input_matches_set_batch():
    x, y = synth.images(40, 3, 20, 20, step=7)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).to(torch.int32).cuda()

    a = _net()
    a.set_batch(xd, yd)
    a.step(0.05, cp.CP_DX_REDUCE_SCATTER, torch.cuda.current_stream(), None, False)
    torch.cuda.synchronize()
    loss_a, par_a = a.loss(), _params(a)
    a.close()

    b = _net()
    sx, sy = torch.empty_like(b.x), torch.empty_like(b.labels)
    sx.copy_(xd.reshape(-1))
    sy.copy_(yd.reshape(-1))
    prev = b.bind_input(sx, sy)
    b.step(0.05, cp.CP_DX_REDUCE_SCATTER, torch.cuda.current_stream(), None, False)
    torch.cuda.synchronize()
    assert b.x.data_ptr() == sx.data_ptr() and b.labels.data_ptr() == sy.data_ptr()
    loss_b, par_b = b.loss(), _params(b)
    back = b.bind_input(*prev)
    assert back[0].data_ptr() == sx.data_ptr()
    b.close()

    assert loss_a == loss_b
    for p, q in zip(par_a, par_b):
        assert torch.equal(p, q)


def test_graph_follows_bound_buffer():
    pn = _net()
    sx, sy = torch.empty_like(pn.x), torch.empty_like(pn.labels)
    prev = pn.bind_input(sx, sy)
    x1, y1 = synth.images(40, 3, 20, 20, step=11)
    sx.copy_(torch.from_numpy(x1).reshape(-1).cuda())
    sy.copy_(torch.from_numpy(y1).to(torch.int32).cuda())
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pn.forward(stream=s)      # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pn.forward(stream=torch.cuda.current_stream())
    pn.bind_input(*prev)
    # new contents in the staging buffer, then replay: the graph reads them
    x2, y2 = synth.images(40, 3, 20, 20, step=12)
    sx.copy_(torch.from_numpy(x2).reshape(-1).cuda())
    sy.copy_(torch.from_numpy(y2).to(torch.int32).cuda())
    g.replay()
    torch.cuda.synchronize()
    loss_graph = pn.loss()
    # eager forward on the same batch through the network's own input
    pn.set_batch(torch.from_numpy(x2).cuda(), torch.from_numpy(y2).to(torch.int32).cuda())
    pn.forward()
    torch.cuda.synchronize()
    assert pn.loss() == loss_graph
    del g
    pn.close()


def test_bind_input_rejects_bad_buffers():
    pn = _net()
    with pytest.raises(ValueError):
        pn.bind_input(torch.empty(7, device="cuda"), torch.empty_like(pn.labels))
    with pytest.raises(ValueError):
        pn.bind_input(torch.empty_like(pn.x), torch.empty(pn.labels.numel(), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        pn.bind_input(torch.empty_like(pn.x, dtype=torch.float64), torch.empty_like(pn.labels))
    pn.close()
