"""A full GCN layer on top of the aggregation SpMM.

    X^{l+1} = sigma(A' (X^l W^l) + b)          (GCNConv; sigma = ReLU here)

Every step runs in libagcn (no cuBLAS): the dense product X W on the tcgen05 tensor cores
(agcn_gemm_xw_ex: TMA + tcgen05.mma + TMEM epilogue) -- precision="fp32" (default) splits both
operands into TF32 high and low parts and accumulates x_hi w_hi + x_lo w_hi + x_hi w_lo
("3xTF32", fp32 accuracy; column slices of W for the widest shapes, a CUDA-core FFMA kernel
for output widths that are not a tcgen05 N), precision="tf32" feeds the operands as TF32; the aggregation, the bias and the
ReLU are the SpMM's fused epilogue or the GEMM's.  The order follows the smaller feature width
(P:124 computes A'(XW); (A'X)W is the same product):

  * F_out <= F_in:  T = X W  (n_cols x F_out), then Y = relu(A T + b)  -- bias + ReLU fused
    into the SpMM's row stores;
  * F_out >  F_in:  T = A X  (n x F_in, SpMM), then Y = relu(T W + b)  -- fused into the GEMM.

Backward uses the same pieces with A^T (``transpose`` / ``gather_vals``).
"""
from __future__ import annotations

from . import Plan, gemm_xw


class GCNLayer:
    """One GCN layer over a plan of A (and optionally of A^T for the backward pass)."""

    def __init__(self, plan: Plan, vals, W, bias=None, relu: bool = True, kernel: str = "auto",
                 precision: str = "fp32"):
        """precision: "fp32" (X W with fp32 accuracy: 3xTF32 on tcgen05, agcn_gemm_xw_ex) or "tf32"
        (TF32 operands, fp32 accumulation).  F_in, F_out in [4, 256], multiples of 4 (tf32: F_out in
        {16, ..., 256})."""
        self.plan, self.vals, self.W, self.bias, self.relu, self.kernel = plan, vals, W, bias, relu, kernel
        self.f_in, self.f_out = int(W.shape[0]), int(W.shape[1])
        if precision not in ("fp32", "tf32"):
            raise ValueError(precision)
        self.precision = precision
        self.Wt = W.t().contiguous()   # K-major B operand

    @property
    def order(self) -> str:
        """'A(XW)' when the output is not wider than the input, else '(AX)W'."""
        return "A(XW)" if self.f_out <= self.f_in else "(AX)W"

    def forward(self, X, out=None, stream=None):
        if X.shape[1] != self.f_in:
            raise ValueError(f"X must have {self.f_in} columns")
        if self.order == "A(XW)":
            T = gemm_xw(X, self.Wt, stream=stream, precision=self.precision)
            return self.plan.spmm(self.vals, T, out=out, stream=stream, kernel=self.kernel,
                                  bias=self.bias, relu=self.relu)
        T = self.plan.spmm(self.vals, X, stream=stream, kernel=self.kernel)
        # bias + ReLU fused into the GEMM epilogue
        return gemm_xw(T, self.Wt, bias=self.bias, relu=self.relu, out=out, stream=stream,
                       precision=self.precision)

    __call__ = forward
