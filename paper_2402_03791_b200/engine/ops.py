"""Tensor-level wrappers over the libzpp C ABI.

torch tensors are used only as device-memory handles (``data_ptr``) and for
stream plumbing; every operation below is one of our sm_100a kernels.
"""

from __future__ import annotations

import torch

from . import lib
from .lib import EPI_BF16, EPI_BF16_DGELU, EPI_BF16_GELU, EPI_F32, EPI_F32_ACC  # noqa: F401


class _Profile:
    """Counts libzpp kernel launches and times every GEMM launch with CUDA events
    on its own stream (bench.py's live roofline, 'gpu_launches')."""

    def __init__(self):
        self.active = False
        self.time_gemms = True
        self.launches = 0
        self._gemms: list = []
        self.shapes: list | None = None   # set to [] to log (M, N, K, algorithmic bytes) per GEMM

    def start(self, time_gemms: bool = True) -> None:
        self.active, self.launches, self._gemms = True, 0, []
        self.time_gemms = time_gemms

    def stop(self, by_shape: bool = False):
        """-> (total GEMM FLOPs, summed GEMM launch ms, GEMM launches); synchronizes.  With
        ``by_shape`` also {(M, N, K, a_t, b_t, epilogue): [launches, FLOPs, ms]}."""
        torch.cuda.synchronize()
        self.active = False
        flops = sum(g[0] for g in self._gemms)
        ms = sum(g[1].elapsed_time(g[2]) for g in self._gemms)
        n = len(self._gemms)
        shapes: dict = {}
        if by_shape:
            for f, a, b, key in self._gemms:
                row = shapes.setdefault(key, [0, 0.0, 0.0])
                row[0] += 1
                row[1] += f
                row[2] += a.elapsed_time(b)
        self._gemms = []
        return (flops, ms, n, shapes) if by_shape else (flops, ms, n)


PROFILE = _Profile()


def _count(n: int) -> None:
    if PROFILE.active:
        PROFILE.launches += n


def _s(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def _p(t) -> int:
    return 0 if t is None else t.data_ptr()


def _ld(t: torch.Tensor) -> int:
    assert t.dim() == 2 and t.stride(1) == 1, "2-D row-major (unit inner stride) tensor expected"
    return t.stride(0)


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, *, a_t: bool = False, b_t: bool = False,
         epilogue: int = EPI_BF16, bias=None, resid=None, aux=None, stream=None) -> torch.Tensor:
    """c[M,N] (op)= A @ B^T with A = a (M x K) or a^T (a is K x M, ``a_t``),
    B = b (N x K) or b^T (b is K x N, ``b_t``)."""
    M = a.shape[1] if a_t else a.shape[0]
    K = a.shape[0] if a_t else a.shape[1]
    N = b.shape[1] if b_t else b.shape[0]
    assert (b.shape[0] if b_t else b.shape[1]) == K, "inner dimensions differ"
    assert c.shape[0] == M and c.shape[1] == N
    sid = _s(stream)
    timed = PROFILE.active and PROFILE.time_gemms
    if timed:
        ts = torch.cuda.ExternalStream(sid)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(ts)
    lib.call("zpp_gemm", _p(a), int(a_t), _ld(a), _p(b), int(b_t), _ld(b), _p(c), _ld(c), M, N, K,
             epilogue, _p(bias), _p(resid), _ld(resid) if resid is not None else 0,
             _p(aux), _ld(aux) if aux is not None else 0, sid)
    if timed:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(ts)
        PROFILE._gemms.append((2.0 * M * N * K, e0, e1, (M, N, K, int(a_t), int(b_t), epilogue)))
    if PROFILE.shapes is not None:
        out_bytes = c.element_size() * (2 if epilogue == EPI_F32_ACC else 1)
        extra = (resid is not None) + (aux is not None)  # residual read; GeLU pre-act write / dGeLU read
        PROFILE.shapes.append((M, N, K, 2 * (M * K + N * K) + M * N * (out_bytes + 2 * extra)))
    _count(1)
    return c


def set_cta_group(cg: int) -> None:
    """GEMM tile policy: 0 auto (CTA pairs when M > 256), 1 single-CTA, 2 prefer pairs."""
    lib.call("zpp_gemm_set_cta_group", cg)


def set_streamk(on: bool) -> None:
    """Enable / disable the stream-K split of the GEMM's last partial wave."""
    lib.call("zpp_gemm_set_streamk", int(on))


def preload() -> None:
    """Load every kernel and allocate the GEMM stream-K workspaces (idempotent)."""
    lib.call("zpp_preload_kernels")


def layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    _count(1)
    lib.call("zpp_layernorm_fwd", _p(x), _p(gamma), _p(beta), _p(y), _p(mean), _p(rstd), rows, cols,
             eps, _s(stream))


def layernorm_bwd_workspace(rows: int, cols: int) -> int:
    return lib.load().zpp_layernorm_bwd_workspace_floats(rows, cols)


def layernorm_bwd(dy, x, mean, rstd, gamma, dx, dgamma, dbeta, workspace, dresid=None, accumulate=True,
                  stream=None):
    """dgamma/dbeta += column sums, or = when ``accumulate`` is False (first writer)."""
    rows, cols = x.shape
    _count(1 if dgamma is None else 2)
    lib.call("zpp_layernorm_bwd", _p(dy), _p(x), _p(mean), _p(rstd), _p(gamma), _p(dresid), _p(dx),
             _p(dgamma), _p(dbeta), _p(workspace), rows, cols, int(accumulate), _s(stream))


def norm_param_grads(dy, x, mean, rstd, dgamma, dbeta, workspace, accumulate=True, stream=None):
    """LayerNorm (mean given) / RMSNorm (mean None) gamma / beta grads alone; pairs with
    layernorm_bwd / rmsnorm_bwd called with dgamma=None."""
    rows, cols = x.shape
    _count(1)
    lib.call("zpp_norm_param_grads", _p(dy), _p(x), _p(mean), _p(rstd), _p(dgamma), _p(dbeta), _p(workspace),
             rows, cols, int(accumulate), _s(stream))


def rmsnorm_fwd(x, gamma, y, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    _count(1)
    lib.call("zpp_rmsnorm_fwd", _p(x), _p(gamma), _p(y), _p(rstd), rows, cols, eps, _s(stream))


def rmsnorm_bwd(dy, x, rstd, gamma, dx, dgamma, workspace, dresid=None, accumulate=True, stream=None):
    """dgamma += column sums of dy * xhat, or = when ``accumulate`` is False (first writer)."""
    rows, cols = x.shape
    _count(1 if dgamma is None else 2)
    lib.call("zpp_rmsnorm_bwd", _p(dy), _p(x), _p(rstd), _p(gamma), _p(dresid), _p(dx), _p(dgamma),
             _p(workspace), rows, cols, int(accumulate), _s(stream))


def swiglu_fwd(gu, a, stream=None):
    rows, ffn = a.shape
    assert gu.shape == (rows, 2 * ffn)
    _count(1)
    lib.call("zpp_swiglu_fwd", _p(gu), _p(a), rows, ffn, _s(stream))


def swiglu_bwd(da, gu, dgu, stream=None):
    rows, ffn = da.shape
    assert gu.shape == dgu.shape == (rows, 2 * ffn)
    _count(1)
    lib.call("zpp_swiglu_bwd", _p(da), _p(gu), _p(dgu), rows, ffn, _s(stream))


def rope(qkv, seq, heads, head_dim, base=10000.0, inverse=False, stream=None):
    """In-place rotary embedding of the q and k parts of qkv [tokens, 3*heads*head_dim]."""
    _count(1)
    lib.call("zpp_rope", _p(qkv), qkv.shape[0], seq, heads, head_dim, base, int(inverse), _s(stream))


def colsum_acc(dy, dbias, workspace, accumulate=True, stream=None):
    rows, cols = dy.shape
    _count(1)
    lib.call("zpp_colsum_acc", _p(dy), _ld(dy), _p(dbias), _p(workspace), rows, cols, int(accumulate),
             _s(stream))


def colsum_workspace(rows: int, cols: int) -> int:
    """Floats of the (zero-initialised, reusable) column-reduction workspace."""
    return layernorm_bwd_workspace(rows, cols)


def gelu(u, g, stream=None):
    _count(1)
    lib.call("zpp_gelu_fwd", _p(u), _p(g), u.numel(), _s(stream))


def attn_fwd(qkv, out, lse, batch, seq, heads, head_dim, stream=None):
    _count(1)
    lib.call("zpp_attn_fwd", _p(qkv), _p(out), _p(lse), batch, seq, heads, head_dim, _s(stream))


def attn_bwd_workspace(batch, seq, heads, head_dim) -> int:
    return lib.load().zpp_attn_bwd_workspace_floats(batch, seq, heads, head_dim)


def attn_bwd(qkv, out, lse, dout, dqkv, workspace, batch, seq, heads, head_dim, stream=None):
    """dQ kernel (also writes delta = rowsum(O dO) and lse*log2e into ``workspace``), then the
    dK/dV kernel; deterministic (no atomics)."""
    _count(2)
    lib.call("zpp_attn_bwd", _p(qkv), _p(out), _p(lse), _p(dout), _p(dqkv), _p(workspace), batch, seq,
             heads, head_dim, _s(stream))


def embed_fwd(ids, wte, wpe, out, seq, stream=None):
    tokens, hidden = out.shape
    _count(1)
    lib.call("zpp_embed_fwd", _p(ids), _p(wte), _p(wpe), _p(out), tokens, seq, hidden, _s(stream))


def embed_bwd(ids, dout, dwte, dwpe, seq, stream=None):
    tokens, hidden = dout.shape
    _count(2 if dwpe is not None else 1)
    lib.call("zpp_embed_bwd", _p(ids), _p(dout), _p(dwte), _p(dwpe), tokens, seq, hidden, dwte.shape[0],
             _s(stream))


def xent(logits, labels, loss_sum, grad_scale, stream=None):
    rows, vocab = logits.shape
    _count(1)
    lib.call("zpp_xent_fwd_bwd", _p(logits), _ld(logits), _p(labels), _p(loss_sum), rows, vocab,
             grad_scale, _s(stream))


def cast_scale(src_f32, dst_bf16, scale=1.0, stream=None):
    if src_f32.numel() != dst_bf16.numel():
        raise ValueError("cast_scale: size mismatch")
    _count(1)
    lib.call("zpp_cast_scale_f32_bf16", _p(src_f32), _p(dst_bf16), src_f32.numel(), scale, _s(stream))


def accum(src_bf16, acc_f32, stream=None):
    if src_bf16.numel() != acc_f32.numel():
        raise ValueError("accum: size mismatch")
    _count(1)
    lib.call("zpp_accum_bf16_f32", _p(src_bf16), _p(acc_f32), src_bf16.numel(), _s(stream))


def accum_f32(src_f32, acc_f32, stream=None):
    """acc += src (fp32); the fp32-wire reduce-scatter's accumulate."""
    if src_f32.numel() != acc_f32.numel():
        raise ValueError("accum_f32: size mismatch")
    _count(1)
    lib.call("zpp_accum_f32_f32", _p(src_f32), _p(acc_f32), src_f32.numel(), _s(stream))


def adamw(master, m, v, grad, param_bf16, lr, beta1, beta2, eps, wd, step, stream=None):
    n = master.numel()
    if not (m.numel() == v.numel() == grad.numel() == param_bf16.numel() == n):
        raise ValueError("adamw: master / exp_avg / exp_avg_sq / grad / bf16 param sizes differ")
    _count(1)
    lib.call("zpp_adamw", _p(master), _p(m), _p(v), _p(grad), _p(param_bf16), master.numel(), lr, beta1,
             beta2, eps, wd, step, _s(stream))


def init_param(master, param_bf16, seed, offset, mean, std, stream=None):
    _count(1)
    lib.call("zpp_init_param", _p(master), _p(param_bf16), master.numel(), seed, offset, mean, std,
             _s(stream))


def zero(t, stream=None):
    """cudaMemsetAsync(0) of a whole tensor on ``stream`` (no torch fill kernel)."""
    lib.call("zpp_zero", _p(t), t.numel() * t.element_size(), _s(stream))
