"""Randomised family sweep (GPU): seeded random layer shapes — odd channel
counts, ragged planes, strides 1-2, every filter size the families
specialise (1x1, 3x3, 5x5, 7x7) plus generic ones — run through EVERY kernel
family that accepts them, at split 1 and 2 (partial planes and, where the
family has one, the DSMEM cluster reduction).  Each result must be within
tol(K) of the float64 oracle, and results whose split channel ranges agree
must be bitwise identical (the fused engine's summation order is a function
of those ranges only — include/b2conv.h).  Complements the fixed plan cases of
test_gpu_parity.py with shapes nobody picked by hand (tile seams across
images, partial row segments, m- and channel tails, TMA out-of-range fill)."""
import numpy as np
import pytest

import paper_2103_16234_b200 as pk
from paper_2103_16234_b200.sharding import _split_bounds

pytestmark = pytest.mark.gpu


def _random_configs(seed=2026, count=48):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        f = int(rng.choice([1, 1, 3, 3, 3, 5, 7, 2]))
        stride = int(rng.choice([1, 1, 2])) if f != 5 else 1
        pad = f // 2 if f > 1 else 0
        hi = 65 if i % 4 == 0 else 33  # every fourth shape on a larger plane (more tiles, TMA boxes)
        h = int(rng.integers(max(f, 5), hi))
        w = int(rng.integers(max(f, 5), hi))
        c = int(rng.choice([3, 4, 8, 12, 16, 20, 24, 36, 40, 64, 72]))
        m = int(rng.choice([5, 16, 24, 40, 64, 70, 96, 130]))
        n = int(rng.integers(1, 5))
        out.append(pk.ConvConfig(f"r{i}", n=n, c=c, h=h, w=w, m=m, hf=f, wf=f, stride=stride, pad_h=pad, pad_w=pad))
    return out


@pytest.mark.parametrize("cfg", _random_configs(), ids=lambda c: c.name)
def test_random_shape_every_family(cfg):
    import oracle
    import torch

    tol = oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)
    g = torch.Generator(device="cuda").manual_seed(17)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
    by_bounds = {}
    runs = 0
    for fam in pk.matching_families(cfg):
        for splits, reduce in ((1, 0), (2, 1), (2, 2)):
            try:
                layer = pk.ConvLayer(cfg, family=fam, splits=splits, reduce=reduce)
            except pk.InvalidPlan:
                continue
            y = layer(x, w)
            torch.cuda.synchronize()
            a = y.cpu().numpy()
            err = oracle.relative_error(a, ref)
            assert err <= tol, (cfg, layer.family, splits, reduce, err)
            key = _split_bounds(layer, cfg.c)
            prev = by_bounds.setdefault(key, (layer.family, a))
            assert prev[1].tobytes() == a.tobytes(), (cfg, prev[0], layer.family, key)
            runs += 1
    assert runs > 0
