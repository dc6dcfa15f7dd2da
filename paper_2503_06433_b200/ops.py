"""Torch-tensor front end of the C ABI.

Thin wrappers: validate dtype/device/contiguity, pass raw pointers and the
current CUDA stream to libseesaw_b200.so.  PyTorch provides memory and streams
only; every op here runs one of the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import SSB_EPI_NONE, SSB_EPI_RESIDUAL, SSB_EPI_SILU_MUL, call


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _check(t: torch.Tensor, name: str, dtype=torch.bfloat16) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def gemm(
    a: torch.Tensor,
    w: torch.Tensor,
    out: torch.Tensor | None = None,
    residual: torch.Tensor | None = None,
    silu_mul: bool = False,
    block_n: int = 0,
) -> torch.Tensor:
    """out = a @ w.T (+ residual) or silu-mul of interleaved gate/up columns.

    a: [M, K] bf16 (row stride may exceed K), w: [N, K] bf16 weight.
    """
    _check(a, "a")
    _check(w, "w")
    M, K = a.shape
    N, K2 = w.shape
    if K != K2:
        raise ValueError(f"gemm: K mismatch {K} vs {K2}")
    if a.stride(1) != 1 or w.stride(1) != 1:
        raise ValueError("gemm: operands must be K-contiguous")
    n_out = N // 2 if silu_mul else N
    if out is None:
        out = torch.empty((M, n_out), dtype=torch.bfloat16, device=a.device)
    _check(out, "out")
    epi = SSB_EPI_SILU_MUL if silu_mul else (SSB_EPI_RESIDUAL if residual is not None else SSB_EPI_NONE)
    if residual is not None:
        _check(residual, "residual")
    call(
        "ssb_gemm_bf16",
        a.data_ptr(),
        w.data_ptr(),
        out.data_ptr(),
        residual.data_ptr() if residual is not None else None,
        M,
        N,
        K,
        a.stride(0),
        w.stride(0),
        out.stride(0),
        residual.stride(0) if residual is not None else 0,
        epi,
        block_n,
        _stream(),
    )
    return out


def kv_reshard_pack(pool, geometry, block_ids, peers, staging) -> None:
    """pool -> staging for every (peer rectangle, block) — see include/seesaw_b200.h."""
    _kv_reshard("ssb_kv_reshard_pack", pool, geometry, block_ids, peers, staging)


def kv_reshard_unpack(pool, geometry, block_ids, peers, staging) -> None:
    """staging -> pool, the inverse placement of :func:`kv_reshard_pack`."""
    _kv_reshard("ssb_kv_reshard_unpack", pool, geometry, block_ids, peers, staging)


def _kv_reshard(name, pool, geometry, block_ids, peers, staging) -> None:
    if not pool.is_cuda or not staging.is_cuda or not block_ids.is_cuda:
        raise ValueError(f"{name}: pool, staging and block ids must be CUDA tensors")
    if block_ids.dtype != torch.int32:
        raise ValueError(f"{name}: block ids must be int32")
    geo = _lib.KVGeometry(*geometry)
    n = len(peers)
    l0 = _lib.int32_array(p[0] for p in peers)
    nl = _lib.int32_array(p[1] for p in peers)
    h0 = _lib.int32_array(p[2] for p in peers)
    nh = _lib.int32_array(p[3] for p in peers)
    off = _lib.int64_array(p[4] for p in peers)
    call(
        name,
        pool.data_ptr(),
        geo,
        block_ids.data_ptr(),
        block_ids.numel(),
        n,
        ctypes.cast(l0, ctypes.POINTER(ctypes.c_int32)),
        ctypes.cast(nl, ctypes.POINTER(ctypes.c_int32)),
        ctypes.cast(h0, ctypes.POINTER(ctypes.c_int32)),
        ctypes.cast(nh, ctypes.POINTER(ctypes.c_int32)),
        ctypes.cast(off, ctypes.POINTER(ctypes.c_int64)),
        staging.data_ptr(),
        _stream(),
    )


def copy2d_batched(src: torch.Tensor, dst: torch.Tensor, descs: torch.Tensor, total_bytes: int) -> None:
    """Batched strided copy; ``descs`` is a CUDA int64 tensor [n, 6] of
    (src_off, dst_off, src_stride, dst_stride, cum_bytes, rows | row_bytes<<32)."""
    if not (src.is_cuda and dst.is_cuda and descs.is_cuda):
        raise ValueError("copy2d_batched: CUDA tensors required")
    if descs.dtype != torch.int64 or descs.dim() != 2 or descs.shape[1] != 6:
        raise ValueError("copy2d_batched: descs must be int64 [n, 6]")
    call(
        "ssb_copy2d_batched",
        src.data_ptr(),
        dst.data_ptr(),
        descs.data_ptr(),
        descs.shape[0],
        total_bytes,
        _stream(),
    )
