"""The paper's four specialised NoScope CNNs (Coral, Roundabout, Taipei, Amsterdam).

The paper gives only their shape ranges ("2--4 convolutional layers, each with
16--64 channels, at most two fully-connected layers, ... regions of video frames of size
50x50", evaluated at batch 64) and their FP16 aggregate arithmetic
intensities at batch 64 (15.1, 37.9, 51.9, 52.7).  The
reference repo carries no layer lists for them.  These are reconstructions in NoScope's
specialised-model family (Kang et al. 2017: blocks of conv3x3 'same' -> ReLU -> conv3x3
'valid' -> ReLU -> maxpool 2x2, the filter count doubling per block, then one hidden dense
layer and a 2-way output), with (filters, blocks, hidden units) chosen so the aggregate AI
under the reference's x8 padding (shapes.py:187-195, roofline.py:65-72) equals the paper's
figure to within 0.3 (``tests/test_host_cpu.py`` checks it).
"""

from __future__ import annotations

from typing import Dict, Tuple

HW = 50
BATCH = 64
# name -> (filters of the first block, blocks, hidden dense units), paper aggregate AI at b64
ARCH: Dict[str, Tuple[int, int, int]] = {
    "noscope_coral": (16, 1, 128),        # AI 15.1
    "noscope_roundabout": (32, 2, 512),   # AI 37.9
    "noscope_taipei": (64, 1, 128),       # AI 51.9
    "noscope_amsterdam": (64, 1, 256),    # AI 52.7
}
PAPER_AI = {"noscope_coral": 15.1, "noscope_roundabout": 37.9, "noscope_taipei": 51.9, "noscope_amsterdam": 52.7}


def build(name: str, seed: int = 0):
    """The torch module (eval mode, seeded random weights): ``features`` (Conv2d / ReLU /
    MaxPool2d) and ``classifier`` (Linear / ReLU / Linear), the VGG layout the protected
    network runner walks."""
    import torch
    import torch.nn as nn

    if name not in ARCH:
        raise ValueError(f"unknown NoScope network {name!r}; expected one of {tuple(ARCH)}")
    filters, blocks, hidden = ARCH[name]
    torch.manual_seed(seed)
    feats, c, h, f = [], 3, HW, filters
    for _ in range(blocks):
        feats += [nn.Conv2d(c, f, 3, padding=1), nn.ReLU(inplace=True), nn.Conv2d(f, f, 3), nn.ReLU(inplace=True),
                  nn.MaxPool2d(2)]
        c, h, f = f, (h - 2) // 2, 2 * f

    class NoScopeCNN(nn.Module):
        def __init__(self):
            super().__init__()
            self.features = nn.Sequential(*feats)
            self.classifier = nn.Sequential(nn.Linear(c * h * h, hidden), nn.ReLU(inplace=True), nn.Linear(hidden, 2))

        def forward(self, x):
            return self.classifier(torch.flatten(self.features(x), 1))
    return NoScopeCNN().eval()
