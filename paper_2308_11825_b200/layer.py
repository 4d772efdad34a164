"""A full GCN layer on top of the aggregation SpMM.

    X^{l+1} = sigma(A' (X^l W^l) + b)          (GCNConv; sigma = ReLU here)

The dense product X W runs either in cuBLAS (precision="fp32": torch.mm with TF32 off, the
same arithmetic class as the SpMM) or on the tcgen05 tensor cores of libagcn
(precision="tf32": agcn_gemm_xw, TMA + tcgen05.mma kind::tf32 + TMEM epilogue); the
aggregation, the bias and the ReLU run in libagcn (agcn_spmm_ex with its fused epilogue).  The order follows the smaller feature width
(P:124 computes A'(XW); (A'X)W is the same product):

  * F_out <= F_in:  T = X W  (n_cols x F_out), then Y = relu(A T + b)  -- bias + ReLU fused
    into the SpMM's row stores;
  * F_out >  F_in:  T = A X  (n x F_in, SpMM), then Y = relu(T W + b)  -- cuBLAS addmm.

Backward uses the same pieces with A^T (``transpose`` / ``gather_vals``).
"""
from __future__ import annotations

from . import Plan, gemm_xw


class GCNLayer:
    """One GCN layer over a plan of A (and optionally of A^T for the backward pass)."""

    def __init__(self, plan: Plan, vals, W, bias=None, relu: bool = True, kernel: str = "auto",
                 precision: str = "fp32"):
        """precision: "fp32" (X W in cuBLAS fp32) or "tf32" (X W on the tcgen05 tensor cores,
        agcn_gemm_xw: TF32 operands, fp32 accumulation; F_out in {16,...,256}, F_in <= 256)."""
        self.plan, self.vals, self.W, self.bias, self.relu, self.kernel = plan, vals, W, bias, relu, kernel
        self.f_in, self.f_out = int(W.shape[0]), int(W.shape[1])
        if precision not in ("fp32", "tf32"):
            raise ValueError(precision)
        self.precision = precision
        self.Wt = W.t().contiguous() if precision == "tf32" else None   # K-major B operand

    @property
    def order(self) -> str:
        """'A(XW)' when the output is not wider than the input, else '(AX)W'."""
        return "A(XW)" if self.f_out <= self.f_in else "(AX)W"

    def forward(self, X, out=None, stream=None):
        import torch
        if X.shape[1] != self.f_in:
            raise ValueError(f"X must have {self.f_in} columns")
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False   # fp32 GEMM (like the SpMM)
        try:
            if self.order == "A(XW)":
                T = gemm_xw(X, self.Wt) if self.precision == "tf32" else torch.mm(X, self.W)
                return self.plan.spmm(self.vals, T, out=out, stream=stream, kernel=self.kernel,
                                      bias=self.bias, relu=self.relu)
            T = self.plan.spmm(self.vals, X, stream=stream, kernel=self.kernel)
            if self.precision == "tf32":  # bias + ReLU fused into the GEMM epilogue
                Y = gemm_xw(T, self.Wt, bias=self.bias, relu=self.relu)
            else:
                Y = torch.addmm(self.bias, T, self.W) if self.bias is not None else torch.mm(T, self.W)
                if self.relu:
                    Y.relu_()
            if out is not None:
                out.copy_(Y)
                return out
            return Y
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    __call__ = forward
