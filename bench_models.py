"""Benchmark workloads (BASELINE.json configs) -- bench support, not product code.

* resnet50     torchvision ResNet-50, 3x224x224, 1000 classes (config 3, the headline)
* resnet32     He et al. 2016 CIFAR ResNet-32 with option-A (parameter-free) shortcuts,
               3x32x32, 10 classes: 31 convs + fc = 32 preconditioned layers (config 2)
* densenet201  torchvision DenseNet-201, 3x224x224 (config 4)
* mlp          784-512-256-10 ReLU MLP with biases (config 1)
Inception-v4 (config 5) has no definition in this image (no timm, not in torchvision).
"""

from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F


class _ShortcutA(nn.Module):
    def __init__(self, planes):
        super().__init__()
        self.pad = planes // 4

    def forward(self, x):
        return F.pad(x[:, :, ::2, ::2], (0, 0, 0, 0, self.pad, self.pad))


class _Basic(nn.Module):
    def __init__(self, inp, planes, stride):
        super().__init__()
        self.conv1 = nn.Conv2d(inp, planes, 3, stride, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(planes)
        self.conv2 = nn.Conv2d(planes, planes, 3, 1, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(planes)
        self.short = _ShortcutA(planes) if (stride != 1 or inp != planes) else nn.Identity()

    def forward(self, x):
        out = F.relu(self.bn1(self.conv1(x)))
        out = self.bn2(self.conv2(out))
        return F.relu(out + self.short(x))


class ResNetCifar(nn.Module):
    def __init__(self, depth=32, classes=10):
        super().__init__()
        n = (depth - 2) // 6
        self.conv1 = nn.Conv2d(3, 16, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(16)
        layers, inp = [], 16
        for planes, stride in ((16, 1), (32, 2), (64, 2)):
            for i in range(n):
                layers.append(_Basic(inp, planes, stride if i == 0 else 1))
                inp = planes
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(64, classes)

    def forward(self, x):
        x = F.relu(self.bn1(self.conv1(x)))
        x = self.layers(x)
        x = F.adaptive_avg_pool2d(x, 1).flatten(1)
        return self.fc(x)


def mlp():
    return nn.Sequential(nn.Flatten(), nn.Linear(784, 512), nn.ReLU(), nn.Linear(512, 256), nn.ReLU(),
                         nn.Linear(256, 10))


WORKLOADS = {
    # name: (constructor, per-GPU batch, input shape, classes)
    "resnet50": (lambda: __import__("torchvision").models.resnet50(), 32, (3, 224, 224), 1000),
    "resnet32": (lambda: ResNetCifar(32, 10), 128, (3, 32, 32), 10),
    "densenet201": (lambda: __import__("torchvision").models.densenet201(), 16, (3, 224, 224), 1000),
    "mlp": (mlp, 64, (1, 28, 28), 10),
}


def layer_geometry(model: nn.Module, in_shape, batch: int):
    """(name, d_in incl. bias, d_out, M, conv geometry or None) for every Linear /
    Conv2d in named_modules() order, via a shape-only forward on the meta device."""
    import copy
    rec = {}
    m = copy.deepcopy(model).to("meta")
    hooks = []
    for name, mod in m.named_modules():
        if isinstance(mod, (nn.Linear, nn.Conv2d)):
            def pre(mod, inp, name=name):
                rec[name] = tuple(inp[0].shape)
            hooks.append(mod.register_forward_pre_hook(pre))
    with torch.no_grad():
        m(torch.empty(batch, *in_shape, device="meta"))
    for h in hooks:
        h.remove()
    out = []
    for name, mod in model.named_modules():
        if isinstance(mod, nn.Conv2d) and mod.groups == 1:
            n, c, h, w = rec[name]
            kh, kw = mod.kernel_size
            oh = (h + 2 * mod.padding[0] - mod.dilation[0] * (kh - 1) - 1) // mod.stride[0] + 1
            ow = (w + 2 * mod.padding[1] - mod.dilation[1] * (kw - 1) - 1) // mod.stride[1] + 1
            bias = mod.bias is not None
            out.append((name, c * kh * kw + int(bias), mod.out_channels, n * oh * ow,
                        dict(shape=(n, c, h, w), k=kh, s=mod.stride[0], p=mod.padding[0], bias=bias)))
        elif isinstance(mod, nn.Linear):
            shp = rec[name]
            mcols = 1
            for s in shp[:-1]:
                mcols *= s
            bias = mod.bias is not None
            out.append((name, mod.in_features + int(bias), mod.out_features, mcols, None))
    return out
