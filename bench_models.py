"""Benchmark workloads (BASELINE.json configs) -- bench support, not product code.

* resnet50     torchvision ResNet-50, 3x224x224, 1000 classes (config 3, the headline)
* resnet32     He et al. 2016 CIFAR ResNet-32 with option-A (parameter-free) shortcuts,
               3x32x32, 10 classes: 31 convs + fc = 32 preconditioned layers (config 2)
* densenet201  torchvision DenseNet-201, 3x224x224 (config 4)
* inception_v4 Szegedy et al. 2016 ("Inception-v4, Inception-ResNet and the Impact of
               Residual Connections", Fig. 9 and Figs. 3-8), 3x299x299, 1000 classes
               (config 5): written here -- no timm in the image and torchvision only
               ships Inception-v3.  149 conv layers + fc; its 1x7/7x1 and 1x3/3x1 convs
               have kh != kw and asymmetric padding (0,3)/(3,0), (0,1)/(1,0).
* mlp          784-512-256-10 ReLU MLP with biases (config 1)
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


class _BC(nn.Module):
    """conv (no bias) + batch-norm + ReLU, the paper's basic unit."""

    def __init__(self, inp, out, k, s=1, p=0):
        super().__init__()
        self.conv = nn.Conv2d(inp, out, k, s, p, bias=False)
        self.bn = nn.BatchNorm2d(out, eps=1e-3)

    def forward(self, x):
        return F.relu(self.bn(self.conv(x)))


class _Cat(nn.Module):
    def __init__(self, *branches):
        super().__init__()
        self.b = nn.ModuleList(branches)

    def forward(self, x):
        return torch.cat([b(x) for b in self.b], 1)


class _Pool(nn.Module):
    def __init__(self, kind, k, s, p=0):
        super().__init__()
        self.kind, self.k, self.s, self.p = kind, k, s, p

    def forward(self, x):
        if self.kind == "max":
            return F.max_pool2d(x, self.k, self.s, self.p)
        return F.avg_pool2d(x, self.k, self.s, self.p, count_include_pad=False)


def _seq(*m):
    return nn.Sequential(*m)


class InceptionV4(nn.Module):
    """Inception-v4 (Szegedy et al. 2016, Fig. 9): stem (Fig. 3), 4 x Inception-A
    (Fig. 4), Reduction-A (Fig. 7, k=192 l=224 m=256 n=384), 7 x Inception-B (Fig. 5),
    Reduction-B (Fig. 8), 3 x Inception-C (Fig. 6), average pool, dropout, fc."""

    def __init__(self, classes=1000):
        super().__init__()
        stem = [_BC(3, 32, 3, 2), _BC(32, 32, 3), _BC(32, 64, 3, p=1),
                _Cat(_Pool("max", 3, 2), _BC(64, 96, 3, 2)),                                   # 160
                _Cat(_seq(_BC(160, 64, 1), _BC(64, 96, 3)),
                     _seq(_BC(160, 64, 1), _BC(64, 64, (7, 1), p=(3, 0)), _BC(64, 64, (1, 7), p=(0, 3)),
                          _BC(64, 96, 3))),                                                    # 192
                _Cat(_BC(192, 192, 3, 2), _Pool("max", 3, 2))]                                 # 384
        blocks = [self._a() for _ in range(4)]
        blocks.append(_Cat(_BC(384, 384, 3, 2),
                           _seq(_BC(384, 192, 1), _BC(192, 224, 3, p=1), _BC(224, 256, 3, 2)),
                           _Pool("max", 3, 2)))                                                # 1024
        blocks += [self._b() for _ in range(7)]
        blocks.append(_Cat(_seq(_BC(1024, 192, 1), _BC(192, 192, 3, 2)),
                           _seq(_BC(1024, 256, 1), _BC(256, 256, (1, 7), p=(0, 3)),
                                _BC(256, 320, (7, 1), p=(3, 0)), _BC(320, 320, 3, 2)),
                           _Pool("max", 3, 2)))                                                # 1536
        blocks += [_InceptionC() for _ in range(3)]
        self.features = nn.Sequential(*stem, *blocks)
        self.fc = nn.Linear(1536, classes)

    @staticmethod
    def _a():
        return _Cat(_seq(_Pool("avg", 3, 1, 1), _BC(384, 96, 1)), _BC(384, 96, 1),
                    _seq(_BC(384, 64, 1), _BC(64, 96, 3, p=1)),
                    _seq(_BC(384, 64, 1), _BC(64, 96, 3, p=1), _BC(96, 96, 3, p=1)))

    @staticmethod
    def _b():
        return _Cat(_seq(_Pool("avg", 3, 1, 1), _BC(1024, 128, 1)), _BC(1024, 384, 1),
                    _seq(_BC(1024, 192, 1), _BC(192, 224, (1, 7), p=(0, 3)), _BC(224, 256, (7, 1), p=(3, 0))),
                    _seq(_BC(1024, 192, 1), _BC(192, 192, (1, 7), p=(0, 3)), _BC(192, 224, (7, 1), p=(3, 0)),
                         _BC(224, 224, (1, 7), p=(0, 3)), _BC(224, 256, (7, 1), p=(3, 0))))

    def forward(self, x):
        x = self.features(x)
        x = F.dropout(F.adaptive_avg_pool2d(x, 1).flatten(1), 0.2, self.training)
        return self.fc(x)


class _InceptionC(nn.Module):
    """Fig. 6: the 1x3 / 3x1 pairs branch off a shared 1x1 (concatenated, 1536 out)."""

    def __init__(self):
        super().__init__()
        self.pool = _seq(_Pool("avg", 3, 1, 1), _BC(1536, 256, 1))
        self.b1 = _BC(1536, 256, 1)
        self.b2 = _BC(1536, 384, 1)
        self.b2a = _BC(384, 256, (1, 3), p=(0, 1))
        self.b2b = _BC(384, 256, (3, 1), p=(1, 0))
        self.b3 = _seq(_BC(1536, 384, 1), _BC(384, 448, (3, 1), p=(1, 0)), _BC(448, 512, (1, 3), p=(0, 1)))
        self.b3a = _BC(512, 256, (1, 3), p=(0, 1))
        self.b3b = _BC(512, 256, (3, 1), p=(1, 0))

    def forward(self, x):
        y2 = self.b2(x)
        y3 = self.b3(x)
        return torch.cat([self.pool(x), self.b1(x), self.b2a(y2), self.b2b(y2), self.b3a(y3), self.b3b(y3)], 1)


def mlp():
    return nn.Sequential(nn.Flatten(), nn.Linear(784, 512), nn.ReLU(), nn.Linear(512, 256), nn.ReLU(),
                         nn.Linear(256, 10))


WORKLOADS = {
    # name: (constructor, per-GPU batch, input shape, classes)
    "resnet50": (lambda: __import__("torchvision").models.resnet50(), 32, (3, 224, 224), 1000),
    "resnet32": (lambda: ResNetCifar(32, 10), 128, (3, 32, 32), 10),
    "densenet201": (lambda: __import__("torchvision").models.densenet201(), 16, (3, 224, 224), 1000),
    "inception_v4": (lambda: InceptionV4(1000), 16, (3, 299, 299), 1000),
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
                        dict(shape=(n, c, h, w), k=kh, s=mod.stride[0], p=mod.padding[0], bias=bias,
                             kernel=(kh, kw), stride=tuple(mod.stride), padding=tuple(mod.padding))))
        elif isinstance(mod, nn.Linear):
            shp = rec[name]
            mcols = 1
            for s in shp[:-1]:
                mcols *= s
            bias = mod.bias is not None
            out.append((name, mod.in_features + int(bias), mod.out_features, mcols, None))
    return out
