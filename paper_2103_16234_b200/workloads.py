"""The BASELINE.json configurations as layer lists.

C1  ResNet conv2_x 3x3, N=1 (the reference's CPU-runnable case)
C2  GoogLeNet inception 1x1 layers (36), N in {1, 8, 16, 32}   <- bench headline
C3  AlexNet conv2 + inception 5x5 layers (10), N in {1, ..., 128}
C4  VGG-16 3x3 layers (13), N in {1, 8, 32, 128}
C5  ResNet-50 v1.5 convolutions (53), N = 256 split over 1/2/4/8 GPUs
"""

from __future__ import annotations

from .configs import ConvConfig

# (name, c, h, m, f, stride, pad) with w = h
_C1 = [("res-conv2x-3x3", 64, 56, 64, 3, 1, 1)]

_INCEPTION = [  # module: (C_in, H, [#1x1, #3x3red, #5x5red, poolproj])
    ("3a", 192, 28, (64, 96, 16, 32)), ("3b", 256, 28, (128, 128, 32, 64)),
    ("4a", 480, 14, (192, 96, 16, 64)), ("4b", 512, 14, (160, 112, 24, 64)),
    ("4c", 512, 14, (128, 128, 24, 64)), ("4d", 512, 14, (112, 144, 32, 64)),
    ("4e", 528, 14, (256, 160, 32, 128)), ("5a", 832, 7, (256, 160, 32, 128)),
    ("5b", 832, 7, (384, 192, 48, 128)),
]
_C2 = [(f"{mod}-{kind}", c, h, m, 1, 1, 0)
       for mod, c, h, ms in _INCEPTION
       for kind, m in zip(("1x1", "3x3red", "5x5red", "poolproj"), ms)]

_C3 = [("alexnet-conv2", 96, 27, 256, 5, 1, 2),
       ("incep-3a-5x5", 16, 28, 32, 5, 1, 2), ("incep-3b-5x5", 32, 28, 96, 5, 1, 2),
       ("incep-4a-5x5", 16, 14, 48, 5, 1, 2), ("incep-4b-5x5", 24, 14, 64, 5, 1, 2),
       ("incep-4c-5x5", 24, 14, 64, 5, 1, 2), ("incep-4d-5x5", 32, 14, 64, 5, 1, 2),
       ("incep-4e-5x5", 32, 14, 128, 5, 1, 2), ("incep-5a-5x5", 32, 7, 128, 5, 1, 2),
       ("incep-5b-5x5", 48, 7, 128, 5, 1, 2)]

_VGG = [("vgg1_1", 3, 224, 64), ("vgg1_2", 64, 224, 64), ("vgg2_1", 64, 112, 128), ("vgg2_2", 128, 112, 128),
        ("vgg3_1", 128, 56, 256), ("vgg3_2", 256, 56, 256), ("vgg3_3", 256, 56, 256),
        ("vgg4_1", 256, 28, 512), ("vgg4_2", 512, 28, 512), ("vgg4_3", 512, 28, 512),
        ("vgg5_1", 512, 14, 512), ("vgg5_2", 512, 14, 512), ("vgg5_3", 512, 14, 512)]
_C4 = [(n, c, h, m, 3, 1, 1) for n, c, h, m in _VGG]


def _resnet50():
    layers = [("conv1", 3, 224, 64, 7, 2, 3)]
    c_in, h = 64, 56
    for stage, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3)), start=1):
        out = width * 4
        for b in range(blocks):
            s = 2 if (b == 0 and stage > 1) else 1
            p = f"layer{stage}.{b}"
            layers.append((f"{p}.conv1", c_in, h, width, 1, 1, 0))
            layers.append((f"{p}.conv2", width, h, width, 3, s, 1))  # v1.5: stride on the 3x3
            h2 = (h + 2 - 3) // s + 1
            layers.append((f"{p}.conv3", width, h2, out, 1, 1, 0))
            if b == 0:
                layers.append((f"{p}.downsample", c_in, h, out, 1, s, 0))
            c_in, h = out, h2
    return layers


_C5 = _resnet50()

WORKLOADS = {
    "c1": (_C1, (1,)),
    "c2": (_C2, (1, 8, 16, 32)),
    "c3": (_C3, (1, 8, 16, 32, 64, 128)),
    "c4": (_C4, (1, 8, 32, 128)),
    "c5": (_C5, (256,)),
}

DESCRIPTIONS = {
    "c1": "ResNet conv2_x 3x3 64->64 56x56",
    "c2": "GoogLeNet inception 1x1 convs (36 layers)",
    "c3": "AlexNet conv2 + inception 5x5 convs (10 layers)",
    "c4": "VGG-16 3x3 convs (13 layers)",
    "c5": "ResNet-50 v1.5 convs (53 layers)",
}


def layers(workload: str, n: int) -> list[ConvConfig]:
    table, _ = WORKLOADS[workload]
    return [ConvConfig(name, n=n, c=c, h=h, w=h, m=m, hf=f, wf=f, stride=s, pad_h=p, pad_w=p)
            for name, c, h, m, f, s, p in table]


def schedule(workload: str, cfgs: list[ConvConfig]) -> list[list[int]]:
    """Dataflow order of a workload's layers for one inference step: groups of
    layer indices that are data-independent in the source network and may
    run concurrently, the groups in dependency order.

    C2  the four branch convolutions of a GoogLeNet inception module (1x1,
        3x3reduce, 5x5reduce read the module input; poolproj reads its
        3x3/s1 max-pool) are independent; modules are sequential.
    C5  in the first block of each ResNet stage the projection shortcut
        (downsample) and conv1 both read the block input; all else chains.
    C1, C3, C4  sequential (single layer; layers of different modules; VGG).
    """
    if workload == "c2":
        groups: dict[str, list[int]] = {}
        for i, c in enumerate(cfgs):
            groups.setdefault(c.name.split("-")[0], []).append(i)
        return list(groups.values())
    if workload == "c5":
        out, idx = [], {c.name: i for i, c in enumerate(cfgs)}
        for i, c in enumerate(cfgs):
            if c.name.endswith(".downsample"):
                continue
            grp = [i]
            if c.name.endswith(".conv1"):
                ds = c.name[: -len("conv1")] + "downsample"
                if ds in idx:
                    grp.append(idx[ds])
            out.append(grp)
        return out
    return [[i] for i in range(len(cfgs))]
