"""The PyTorch operator library torch.ops.b2conv (csrc/torch_ext.cpp).

CPU host: the library loads, both operators are registered and their Meta
kernels give F.conv2d's output shapes (fake-tensor tracing never touches a
device).  GPU: the CUDA kernels against the f64 oracle, the out= variant,
concurrent streams (each call takes its scratch from the caching allocator on
its own stream) and torch.compile(fullgraph=True) tracing through the Meta
kernel.  Entry point replaced: convkit.twostage.conv_twostage
(/root/reference/pkg/src/convkit/twostage.py:208-212).
"""

from __future__ import annotations

import pytest
import torch

import paper_2103_16234_b200 as pk
from paper_2103_16234_b200.engine import torch_ops

SHAPES = [((2, 16, 14, 14), (32, 16, 3, 3), 1, (1, 1)), ((1, 3, 224, 224), (64, 3, 7, 7), 2, (3, 3)),
          ((4, 64, 56, 56), (256, 64, 1, 1), 1, (0, 0)), ((2, 8, 9, 7), (5, 8, 2, 4), 3, (1, 2))]


def test_operator_library_registers_conv2d_with_meta_kernels():
    ops = torch_ops()
    for xs, ws, s, p in SHAPES:
        x, w = torch.empty(xs, device="meta"), torch.empty(ws, device="meta")
        want = torch.nn.functional.conv2d(torch.empty(xs, device="meta"), torch.empty(ws, device="meta"),
                                          stride=s, padding=p).shape
        assert ops.conv2d(x, w, [s, s], list(p), "fused").shape == want
        assert ops.conv2d(x, w, [s, s], list(p), "tf32x3").shape == want
        out = torch.empty(want, device="meta")
        assert ops.conv2d_out(x, w, [s, s], list(p), "fused", out=out).shape == want


def test_meta_kernel_rejects_bad_operands():
    ops = torch_ops()
    x, w = torch.empty((2, 16, 14, 14), device="meta"), torch.empty((8, 15, 3, 3), device="meta")
    with pytest.raises(RuntimeError, match="filter depth"):
        ops.conv2d(x, w, [1, 1], [1, 1], "fused")
    with pytest.raises(RuntimeError, match="unknown engine"):
        ops.conv2d(x, torch.empty((8, 16, 3, 3), device="meta"), [1, 1], [1, 1], "winograd")
    with pytest.raises(RuntimeError, match="one stride"):
        ops.conv2d(x, torch.empty((8, 16, 3, 3), device="meta"), [1, 2], [1, 1], "fused")


def test_fake_tensor_tracing_uses_the_meta_kernel():
    from torch._subclasses.fake_tensor import FakeTensorMode

    ops = torch_ops()
    with FakeTensorMode():
        x = torch.empty((2, 16, 14, 14), device="cuda")
        w = torch.empty((32, 16, 3, 3), device="cuda")
        y = ops.conv2d(x, w, [1, 1], [1, 1], "fused")
        assert y.shape == (2, 32, 14, 14) and y.device.type == "cuda"


def _rand(shape, seed):
    import oracle

    return torch.from_numpy(oracle.make_uniform(shape, seed))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["fused", "twostage", "tf32x3"])
def test_operator_matches_oracle(engine):
    import oracle

    for i, (xs, ws, s, p) in enumerate(SHAPES):
        if engine == "twostage" and s != 1:
            continue
        cfg = pk.ConvConfig("op", n=xs[0], c=xs[1], h=xs[2], w=xs[3], m=ws[0], hf=ws[2], wf=ws[3], stride=s,
                            pad_h=p[0], pad_w=p[1])
        xc, wc = _rand(xs, 10 + i), _rand(ws, 20 + i)
        y = torch_ops().conv2d(xc.cuda(), wc.cuda(), [s, s], list(p), engine).cpu().numpy()
        if engine == "twostage":
            assert y.tobytes() == oracle.conv_naive(cfg, xc.numpy(), wc.numpy()).tobytes()
        else:
            ref = oracle.conv_f64(cfg, xc.numpy(), wc.numpy())
            assert oracle.relative_error(y, ref) <= oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)


@pytest.mark.gpu
def test_operator_out_variant_and_public_conv2d_route():
    x, w = _rand((2, 64, 14, 14), 1).cuda(), _rand((48, 64, 3, 3), 2).cuda()
    out = torch.full((2, 48, 14, 14), float("nan"), device="cuda")
    r = torch_ops().conv2d_out(x, w, [1, 1], [1, 1], "fused", out=out)
    assert r.data_ptr() == out.data_ptr()
    y = pk.conv2d(x, w, stride=1, padding=1)  # the public entry dispatches through the operator
    assert torch.equal(y, out)
    with pytest.raises(pk.ShapeMismatch):
        pk.conv2d(x, w, stride=1, padding=1, out=torch.empty((2, 48, 13, 14), device="cuda"))
    with pytest.raises(pk.ShapeMismatch):
        pk.conv2d(x.double(), w.double())


@pytest.mark.gpu
def test_concurrent_streams_same_shape_split_plans():
    """Two streams, same shape, a split-C plan (workspace): each call's
    partial planes come from the caching allocator on its own stream, so the
    results are the single-stream results."""
    x1, w = _rand((4, 512, 7, 7), 3).cuda(), _rand((128, 512, 1, 1), 4).cuda()
    x2 = _rand((4, 512, 7, 7), 5).cuda()
    ops = torch_ops()
    want1, want2 = ops.conv2d(x1, w, [1, 1], [0, 0]), ops.conv2d(x2, w, [1, 1], [0, 0])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(20):
        with torch.cuda.stream(s1):
            a = ops.conv2d(x1, w, [1, 1], [0, 0])
        with torch.cuda.stream(s2):
            b = ops.conv2d(x2, w, [1, 1], [0, 0])
        outs.append((a, b))
    torch.cuda.synchronize()
    for a, b in outs:
        assert torch.equal(a, want1) and torch.equal(b, want2)
    # the same through ConvLayer (workspace keyed by stream)
    layer = pk.ConvLayer(pk.ConvConfig("s", n=4, c=512, h=7, w=7, m=128, hf=1, wf=1), splits=4, reduce=1)
    ref1, ref2 = layer(x1, w), layer(x2, w)
    res = []
    for _ in range(20):
        with torch.cuda.stream(s1):
            a = layer(x1, w)
        with torch.cuda.stream(s2):
            b = layer(x2, w)
        res.append((a, b))
    torch.cuda.synchronize()
    assert all(torch.equal(a, ref1) and torch.equal(b, ref2) for a, b in res)


@pytest.mark.gpu
def test_torch_compile_fullgraph_traces_the_operator():
    import oracle

    ops = torch_ops()

    def block(x, w1, w2):
        y = ops.conv2d(x, w1, [1, 1], [1, 1], "fused")
        return ops.conv2d(y, w2, [2, 2], [0, 0], "fused")

    x, w1, w2 = _rand((2, 16, 14, 14), 7).cuda(), _rand((24, 16, 3, 3), 8).cuda(), _rand((8, 24, 1, 1), 9).cuda()
    eager = block(x, w1, w2)
    for backend in ("aot_eager", "inductor"):
        torch._dynamo.reset()
        compiled = torch.compile(block, fullgraph=True, backend=backend)
        assert torch.equal(compiled(x, w1, w2), eager), backend
    c1 = pk.ConvConfig("a", n=2, c=16, h=14, w=14, m=24, hf=3, wf=3, pad_h=1, pad_w=1)
    c2 = pk.ConvConfig("b", n=2, c=24, h=14, w=14, m=8, hf=1, wf=1, stride=2)
    y1 = oracle.conv_f64(c1, x.cpu().numpy(), w1.cpu().numpy())
    ref = oracle.conv_f64(c2, y1, w2.cpu().numpy())
    assert oracle.relative_error(eager.cpu().numpy(), ref) <= 1e-5
