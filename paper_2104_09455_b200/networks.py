"""Linear-layer lists of the paper's CNN workloads (configs C3-C5), from torchvision.

The reference describes networks only as ``ModelSpec`` layer lists (shapes.py:52-69,
fixtures.py) and the paper measures "a network's overhead as the sum over its linear
layers".  The paper's layer lists are those of the torchvision models:
forward hooks on every Conv2d / Linear of the model on the ``meta`` device give each
layer's input extent, stride and padding (SURVEY Appendix A reproduces Fig 4/5 from
exactly this capture).  Grouped / depthwise convolutions are treated as dense, as the
paper does (documents.py:111-112 rejects groups).

No weights are materialised here: ``LayerSpec`` only carries geometry; the benchmark
creates seeded synthetic weights and activations of these shapes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

from .shapes import GemmShape

NETWORKS = ("resnet50", "vgg16", "alexnet", "squeezenet1_0", "shufflenet_v2_x1_0",
            # the paper's remaining Fig 4 workloads
            "densenet161", "resnext50_32x4d", "wide_resnet50_2",
            # the specialised NoScope CNNs (50x50 frames, batch 64; noscope.py)
            "noscope_coral", "noscope_roundabout", "noscope_taipei", "noscope_amsterdam")


@dataclass(frozen=True)
class LayerSpec:
    """One linear layer as an NHWC convolution (an FC layer is a 1x1 conv on a 1x1 image)."""

    index: int
    kind: str            # "conv" | "fc"
    n: int
    h: int
    w: int
    cin: int
    oc: int
    r: int
    s: int
    stride_h: int
    stride_w: int
    pad_h: int
    pad_w: int

    @property
    def p(self) -> int:
        return (self.h + 2 * self.pad_h - self.r) // self.stride_h + 1

    @property
    def q(self) -> int:
        return (self.w + 2 * self.pad_w - self.s) // self.stride_w + 1

    def gemm(self) -> GemmShape:
        """The reference lowering (shapes.py:169-177): M = n*P*Q, N = OC, K = C*R*S."""
        return GemmShape(self.n * self.p * self.q, self.oc, self.cin * self.r * self.s)


def capture(name: str, batch: int, h: int, w: int) -> List[LayerSpec]:
    """Conv2d / Linear layers of torchvision ``name`` in forward order for a [batch, 3, h, w] input."""
    import torch
    import torchvision

    if name not in NETWORKS:
        raise ValueError(f"unknown network {name!r}; expected one of {NETWORKS}")
    with torch.device("meta"):
        if name.startswith("noscope_"):
            from . import noscope
            model = noscope.build(name)
        else:
            model = getattr(torchvision.models, name)(weights=None)
    model.eval()
    layers: List[LayerSpec] = []

    def hook(mod, inputs, _out):
        x = inputs[0]
        if isinstance(mod, torch.nn.Conv2d):
            nb, c, hh, ww = x.shape
            layers.append(LayerSpec(len(layers), "conv", int(nb), int(hh), int(ww), int(c), mod.out_channels,
                                    mod.kernel_size[0], mod.kernel_size[1], mod.stride[0], mod.stride[1],
                                    mod.padding[0], mod.padding[1]))
        else:
            nb, f = x.shape
            layers.append(LayerSpec(len(layers), "fc", int(nb), 1, 1, int(f), mod.out_features, 1, 1, 1, 1, 0, 0))

    handles = [m.register_forward_hook(hook) for m in model.modules()
               if isinstance(m, (torch.nn.Conv2d, torch.nn.Linear))]
    with torch.no_grad():
        model(torch.empty(batch, 3, h, w, device="meta"))
    for hd in handles:
        hd.remove()
    return layers
