"""KSLinear: a drop-in inference replacement for ``torch.nn.Linear`` whose
weight is a product of Kronecker-sparse factors W = K_1 ... K_L (the paper's
layer).

forward(x) = act(x W^T + bias), computed by ks_chain_bias / ks_chain_act (all
factors on the GPU kernels of libks.so, the bias and the optional GELU -- the
FFN row of Table 7, PAPER.md:1568 -- fused into the last factor's epilogue).  Both
batch layouts are supported: ``layout="bsf"`` takes x of
shape (..., in_features); ``layout="bsl"`` takes x of shape (in_features, B).
Inference only (the paper's scope): no autograd.
"""
from __future__ import annotations

import math

import torch

from . import ks


def _chainable(patterns) -> bool:
    return all(p[0] * p[2] * p[3] == q[0] * q[1] * q[3] for p, q in zip(patterns[:-1], patterns[1:]))


class KSLinear(torch.nn.Module):
    def __init__(self, patterns, weights=None, bias: bool | torch.Tensor = True, layout: str = "bsf",
                 math_mode: str = "fp32", device="cuda", generator: torch.Generator | None = None,
                 activation: str | None = None):
        """patterns: [(a,b,c,d), ...] in product order K_1..K_L (a_l c_l d_l ==
        a_{l+1} b_{l+1} d_{l+1}).  math_mode: "fp32" (CUDA cores),
        "tf32" or "f32x3" (FP32-accurate 3xTF32) on the tensor cores for factors
        with b, c >= 16.  weights: matching list of
        canonical (a,b,c,d) float32 tensors/arrays, or None for the paper's
        initialisation U[-1/sqrt(c), 1/sqrt(c)]."""
        super().__init__()
        ks._act(activation)
        self.activation = activation
        patterns = [tuple(int(v) for v in p) for p in patterns]
        if not patterns or not _chainable(patterns):
            raise ValueError(f"patterns are not a chain: {patterns}")
        self.patterns = patterns
        self.layout = layout
        self.in_features = patterns[-1][0] * patterns[-1][2] * patterns[-1][3]
        self.out_features = patterns[0][0] * patterns[0][1] * patterns[0][3]
        dev = torch.device(device)
        if weights is None:
            weights = []
            for (a, b, c, d) in patterns:
                w = torch.empty((a, b, c, d), dtype=torch.float32)
                w.uniform_(-1.0 / math.sqrt(c), 1.0 / math.sqrt(c), generator=generator)
                weights.append(w)
        self.factors = []
        for p, w in zip(patterns, weights):
            t = torch.as_tensor(w, dtype=torch.float32).contiguous().to(dev)
            f = ks.Factor(*p, t)
            if math_mode in ("tf32", "f32x3") and p[1] >= 16 and p[2] >= 16:
                f.set_math(ks.MATH_TF32 if math_mode == "tf32" else ks.MATH_F32X3)
            self.factors.append(f)
        if isinstance(bias, torch.Tensor):
            if bias.numel() != self.out_features:
                raise ValueError(f"bias must have out_features = {self.out_features} values, got {bias.numel()}")
            self.bias = torch.nn.Parameter(bias.detach().to(dev, torch.float32).contiguous(), requires_grad=False)
        elif bias:
            bound = 1.0 / math.sqrt(self.in_features)
            b = torch.empty(self.out_features, dtype=torch.float32).uniform_(-bound, bound, generator=generator)
            self.bias = torch.nn.Parameter(b.to(dev), requires_grad=False)
        else:
            self.register_parameter("bias", None)

    @torch.no_grad()
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.dtype != torch.float32:
            raise TypeError("KSLinear computes in float32")
        if self.layout == "bsl":
            if x.dim() != 2 or x.shape[0] != self.in_features:
                raise ValueError(f"BSL input must be ({self.in_features}, B)")
            return ks.chain(self.factors, x.contiguous(), layout="bsl", bias=self.bias, act=self.activation)
        lead = x.shape[:-1]
        if x.shape[-1] != self.in_features:
            raise ValueError(f"last dimension must be {self.in_features}")
        x2 = x.reshape(-1, self.in_features).contiguous()
        y = ks.chain(self.factors, x2, layout="bsf", bias=self.bias, act=self.activation)
        return y.reshape(*lead, self.out_features)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"patterns={self.patterns}, layout={self.layout}, bias={self.bias is not None}")
