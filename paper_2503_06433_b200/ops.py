"""Torch-tensor front end of the C ABI.

Thin wrappers: validate dtype/device/contiguity, pass raw pointers and the
current CUDA stream to libseesaw_b200.so.  PyTorch provides memory and streams
only; every op here runs one of the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from ._lib import SSB_EPI_F32, SSB_EPI_NONE, SSB_EPI_RESIDUAL, SSB_EPI_SILU_MUL, call, load


def gemm_plan(M: int, N: int, K: int, epilogue: int = SSB_EPI_NONE, max_ctas: int = 0,
              workspace_bytes: int = 0) -> tuple[tuple[int, int, int], int]:
    """((mode, block_n, splits), workspace bytes) the library picks for a shape."""
    out = (ctypes.c_int32 * 3)()
    need = load().ssb_gemm_plan(M, N, K, epilogue, max_ctas, workspace_bytes, out)
    if need < 0:
        raise ValueError(load().ssb_last_error().decode())
    return (out[0], out[1], out[2]), int(need)


# prefill attention kernel variant for A/B runs (see ssb_prefill_attention)
_PREFILL_VARIANT = int(os.environ.get("SSB_PREFILL_ATTN_VARIANT", "0"))


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
    out_f32: bool = False,
    max_ctas: int = 0,
    workspace: torch.Tensor | None = None,
    rownorm: "_lib.RowNorm | None" = None,
) -> torch.Tensor:
    """out = a @ w.T (+ residual) or silu-mul of interleaved gate/up columns,
    or fp32 output (logits) with ``out_f32``.

    a: [M, K] bf16 (row stride may exceed K), w: [N, K] bf16 weight.
    workspace: zero-initialised device buffer (one per stream) that lets the
    library split K across CTAs for skinny problems (decode projections).
    rownorm: the folded-RMSNorm hooks (row_norm(); ss_parts is filled in).
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
    odt = torch.float32 if out_f32 else torch.bfloat16
    if out is None:
        out = torch.empty((M, n_out), dtype=odt, device=a.device)
    _check(out, "out", odt)
    if out_f32:
        epi = SSB_EPI_F32
    else:
        epi = SSB_EPI_SILU_MUL if silu_mul else (SSB_EPI_RESIDUAL if residual is not None else SSB_EPI_NONE)
    if residual is not None:
        _check(residual, "residual")
    call(
        "ssb_gemm_bf16_rn" if rownorm is not None else "ssb_gemm_bf16_ws",
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
        max_ctas,
        workspace.data_ptr() if workspace is not None else None,
        workspace.numel() * workspace.element_size() if workspace is not None else 0,
        *((ctypes.byref(rownorm),) if rownorm is not None else ()),
        _stream(),
    )
    return out


def row_norm(ss_out: torch.Tensor | None = None, ss_in: torch.Tensor | None = None, ss_in_parts: int = 0,
             hidden: int = 0, eps: float = 0.0) -> "_lib.RowNorm":
    """Folded-RMSNorm hooks of one GEMM (include/seesaw_b200.h ssb_rownorm):
    ``ss_out`` fp32 [M, >= N tiles] receives the producer's per-tile row sums
    of squares (residual epilogue; ``.ss_parts`` = tiles written), ``ss_in``
    (a producer's ss_out, ``ss_in_parts`` columns used) scales every output
    row by 1/rms before the epilogue."""
    for t, n in ((ss_out, "ss_out"), (ss_in, "ss_in")):
        if t is not None and (t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous()):
            raise ValueError(f"row_norm: {n} must be a contiguous fp32 CUDA tensor")
    if ss_in is not None and ss_in.shape[1] != ss_in_parts:
        raise ValueError(f"row_norm: ss_in has {ss_in.shape[1]} columns, ss_in_parts={ss_in_parts}")
    return _lib.RowNorm(ss_out.data_ptr() if ss_out is not None else None,
                        ss_in.data_ptr() if ss_in is not None else None, ss_in_parts, hidden, eps, 0)


def kv_reshard_pack(pool, geometry, block_ids, peers, staging) -> None:
    """pool -> staging for every (peer rectangle, block) — see include/seesaw_b200.h."""
    _kv_reshard("ssb_kv_reshard_pack", pool, geometry, block_ids, peers, staging)


def kv_reshard_unpack(pool, geometry, block_ids, peers, staging) -> None:
    """staging -> pool, the inverse placement of :func:`kv_reshard_pack`."""
    _kv_reshard("ssb_kv_reshard_unpack", pool, geometry, block_ids, peers, staging)


def kv_reshard_pack_p2p(pool, geometry, block_ids, peers) -> None:
    """pool -> every peer's receive buffer directly (peer memory): ``peers``
    are (l0, nl, h0, nh, absolute destination address) per peer."""
    if not pool.is_cuda or not block_ids.is_cuda or block_ids.dtype != torch.int32:
        raise ValueError("kv_reshard_pack_p2p: CUDA pool and int32 CUDA block ids required")
    geo = _lib.KVGeometry(*geometry)
    arrs = [_lib.int32_array(p[i] for p in peers) for i in range(4)]
    dst = _lib.int64_array(p[4] for p in peers)
    call("ssb_kv_reshard_pack_p2p", pool.data_ptr(), geo, block_ids.data_ptr(), block_ids.numel(), len(peers),
         *[ctypes.cast(a, ctypes.POINTER(ctypes.c_int32)) for a in arrs], ctypes.cast(dst, ctypes.POINTER(ctypes.c_int64)),
         _stream())


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


def copy2d_batched(src: torch.Tensor, dst: torch.Tensor | None, descs: torch.Tensor, total_bytes: int) -> None:
    """Batched strided copy; ``descs`` is a CUDA int64 tensor [n, 6] of
    (src_off, dst_off, src_stride, dst_stride, cum_bytes, rows | row_bytes<<32).
    ``dst=None``: dst_off are absolute device addresses (peer memory)."""
    if not (src.is_cuda and (dst is None or dst.is_cuda) and descs.is_cuda):
        raise ValueError("copy2d_batched: CUDA tensors required")
    if descs.dtype != torch.int64 or descs.dim() != 2 or descs.shape[1] != 6:
        raise ValueError("copy2d_batched: descs must be int64 [n, 6]")
    call(
        "ssb_copy2d_batched",
        src.data_ptr(),
        dst.data_ptr() if dst is not None else None,
        descs.data_ptr(),
        descs.shape[0],
        total_bytes,
        _stream(),
    )


def kv_hnd_copy(gather: bool, pool: torch.Tensor, geometry, blocks: torch.Tensor, n_tokens: int,
                rect: tuple[int, int, int, int], staging: torch.Tensor, stream: int | None = None) -> None:
    """One sequence's KV rectangle (l0, nl, h0, nh) between the pool and a
    contiguous HND staging buffer [nl][2][nh][n_tokens][d] (host-tier swap)."""
    if blocks.dtype != torch.int32 or not blocks.is_cuda:
        raise ValueError("kv_hnd_copy: blocks must be a CUDA int32 tensor")
    l0, nl, h0, nh = rect
    call("ssb_kv_hnd_copy", 1 if gather else 0, pool.data_ptr(), _lib.KVGeometry(*geometry), blocks.data_ptr(),
         blocks.numel(), n_tokens, l0, nl, h0, nh, staging.data_ptr(), stream if stream is not None else _stream())


def memcpy2d_async(dst_ptr: int, dpitch: int, src_ptr: int, spitch: int, width: int, height: int,
                   stream: int | None = None) -> None:
    call("ssb_memcpy2d_async", dst_ptr, dpitch, src_ptr, spitch, width, height,
         stream if stream is not None else _stream())


def init_weights(arena: torch.Tensor, segs: torch.Tensor, total_elems: int, seed: int) -> None:
    """Counter-based init of ``arena`` (bf16) from a CUDA int64 [n, 8] segment table."""
    _check(arena, "arena")
    if not segs.is_cuda or segs.dtype != torch.int64 or segs.shape[1] != 8:
        raise ValueError("init_weights: segs must be a CUDA int64 [n, 8] table")
    call("ssb_init_weights", arena.data_ptr(), segs.data_ptr(), segs.shape[0], total_elems, seed, _stream())


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float, out: torch.Tensor | None = None,
            row_idx: torch.Tensor | None = None) -> torch.Tensor:
    """RMSNorm of x's rows (or of the rows listed in int32 ``row_idx``)."""
    _check(x, "x")
    _check(w, "w")
    hidden = x.shape[1]
    rows = row_idx.numel() if row_idx is not None else x.shape[0]
    if row_idx is not None and row_idx.dtype != torch.int32:
        raise ValueError("rmsnorm: row_idx must be int32")
    if out is None:
        out = torch.empty((rows, hidden), dtype=torch.bfloat16, device=x.device)
    call("ssb_rmsnorm", x.data_ptr(), x.stride(0), row_idx.data_ptr() if row_idx is not None else None,
         w.data_ptr(), out.data_ptr(), out.stride(0), rows, hidden, eps, _stream())
    return out


def decode_positions(ctx_lens: torch.Tensor, block_tables: torch.Tensor, block_size: int,
                     positions: torch.Tensor, slots: torch.Tensor) -> None:
    """Advance every context by one token and compute its position and pool slot."""
    call("ssb_decode_positions", ctx_lens.data_ptr(), block_tables.data_ptr(), block_tables.shape[1], block_size,
         positions.data_ptr(), slots.data_ptr(), ctx_lens.numel(), _stream())


def rope_kv_append(qkv: torch.Tensor, nq: int, nk: int, positions: torch.Tensor, rope_cos: torch.Tensor,
                   rope_sin: torch.Tensor, pool: torch.Tensor | None, geometry, layer: int,
                   slots: torch.Tensor | None) -> None:
    """In-place RoPE on q/k heads of ``qkv`` and paged append of k/v (see C ABI)."""
    _check(qkv, "qkv")
    if positions.dtype != torch.int32 or rope_cos.dtype != torch.float32:
        raise ValueError("rope_kv_append: positions int32, tables float32")
    if slots is not None and slots.dtype != torch.int64:
        raise ValueError("rope_kv_append: slots must be int64")
    call("ssb_rope_kv_append", qkv.data_ptr(), qkv.stride(0), qkv.shape[0], nq, nk, positions.data_ptr(),
         rope_cos.data_ptr(), rope_sin.data_ptr(), rope_cos.shape[0],
         pool.data_ptr() if pool is not None else None, _lib.KVGeometry(*geometry), layer,
         slots.data_ptr() if slots is not None else None, _stream())


def gemm_qkv_rope_kv(a: torch.Tensor, w: torch.Tensor, out: torch.Tensor, nq: int, nk: int,
                     positions: torch.Tensor, rope_cos: torch.Tensor, rope_sin: torch.Tensor,
                     pool: torch.Tensor | None, geometry, layer: int, slots: torch.Tensor | None,
                     block_n: int = 0, max_ctas: int = 0, workspace: torch.Tensor | None = None,
                     rownorm: "_lib.RowNorm | None" = None) -> torch.Tensor:
    """QKV projection with RoPE and the paged K/V append fused into the GEMM
    epilogue: bit-identical to gemm() followed by rope_kv_append()."""
    _check(a, "a")
    _check(w, "w")
    _check(out, "out")
    M, K = a.shape
    d = rope_cos.shape[1] * 2
    if w.shape[0] != (nq + 2 * nk) * d or w.shape[1] != K:
        raise ValueError(f"gemm_qkv_rope_kv: weight {tuple(w.shape)} is not [(nq+2nk)*{d}, {K}]")
    if positions.dtype != torch.int32 or rope_cos.dtype != torch.float32:
        raise ValueError("gemm_qkv_rope_kv: positions int32, tables float32")
    if slots is not None and slots.dtype != torch.int64:
        raise ValueError("gemm_qkv_rope_kv: slots must be int64")
    call("ssb_gemm_qkv_rope_kv", a.data_ptr(), w.data_ptr(), out.data_ptr(), M, K, a.stride(0), w.stride(0),
         out.stride(0), nq, nk, d, positions.data_ptr(), rope_cos.data_ptr(), rope_sin.data_ptr(),
         rope_cos.shape[0], pool.data_ptr() if pool is not None else None, _lib.KVGeometry(*geometry), layer,
         slots.data_ptr() if slots is not None else None, block_n, max_ctas,
         workspace.data_ptr() if workspace is not None else None,
         workspace.numel() * workspace.element_size() if workspace is not None else 0,
         ctypes.byref(rownorm) if rownorm is not None else None, _stream())
    return out


def lm_head_argmax(h: torch.Tensor, w: torch.Tensor, index_base: int, out_val: torch.Tensor,
                   out_idx: torch.Tensor, keys: torch.Tensor | None = None,
                   workspace: torch.Tensor | None = None, rownorm: "_lib.RowNorm | None" = None) -> None:
    """Greedy argmax of h @ w.T without materialising the logits: the GEMM
    epilogue reduces each row to a packed (value, index) key (64-bit
    atomicMax), then the keys are unpacked to (value, index + index_base)."""
    _check(h, "h")
    _check(w, "w")
    M, K = h.shape
    N = w.shape[0]
    if keys is None:
        keys = torch.empty(M, dtype=torch.int64, device=h.device)
    call("ssb_gemm_lm_head_argmax", h.data_ptr(), w.data_ptr(), M, N, K, h.stride(0), w.stride(0), index_base,
         keys.data_ptr(), 0, 0, workspace.data_ptr() if workspace is not None else None,
         workspace.numel() * workspace.element_size() if workspace is not None else 0,
         ctypes.byref(rownorm) if rownorm is not None else None, _stream())
    call("ssb_argmax_keys_decode", keys.data_ptr(), M, out_val.data_ptr(), out_idx.data_ptr(), _stream())


def embedding(ids: torch.Tensor, table: torch.Tensor, vocab_begin: int, out: torch.Tensor) -> torch.Tensor:
    _check(table, "table")
    if ids.dtype != torch.int32:
        raise ValueError("embedding: ids must be int32")
    call("ssb_embedding", ids.data_ptr(), ids.numel(), table.data_ptr(), vocab_begin, table.shape[0],
         table.shape[1], out.data_ptr(), out.stride(0), _stream())
    return out


def argmax_rows(logits: torch.Tensor, index_base: int, out_val: torch.Tensor, out_idx: torch.Tensor) -> None:
    _check(logits, "logits", torch.float32)
    rows, cols = logits.shape
    call("ssb_argmax_rows", logits.data_ptr(), logits.stride(0), rows, cols, index_base, out_val.data_ptr(),
         out_idx.data_ptr(), _stream())


def argmax_combine(vals: torch.Tensor, idxs: torch.Tensor, out_idx: torch.Tensor) -> None:
    parts, rows = vals.shape
    call("ssb_argmax_combine", vals.data_ptr(), idxs.data_ptr(), parts, rows, out_idx.data_ptr(), _stream())


def prefill_attention(qkv: torch.Tensor, nq: int, nk: int, head_dim: int, cu_seqlens: torch.Tensor,
                      max_len: int, out: torch.Tensor, scale: float, variant: int | None = None) -> torch.Tensor:
    """Causal varlen attention over packed prompts.  variant 0 (default,
    ``SSB_PREFILL_ATTN_VARIANT``): persistent tcgen05 kernel for head_dim 128
    (two query heads per CTA when the GQA group is even); 1: mma.sync kernel;
    2: tcgen05 kernel with one CTA per (query tile, head, sequence)."""
    if variant is None:  # SSB_PREFILL_ATTN_VARIANT: A/B switch of the kernel variant
        variant = _PREFILL_VARIANT
    _check(qkv, "qkv")
    _check(out, "out")
    if cu_seqlens.dtype != torch.int32:
        raise ValueError("prefill_attention: cu_seqlens must be int32")
    call("ssb_prefill_attention", qkv.data_ptr(), qkv.stride(0), qkv.shape[0], nq, nk, head_dim,
         cu_seqlens.data_ptr(), cu_seqlens.numel() - 1, max_len, out.data_ptr(), out.stride(0), scale, variant,
         _stream())
    return out


def decode_attention(qkv: torch.Tensor, nq: int, nk: int, pool: torch.Tensor, geometry, num_blocks: int,
                     layer: int, block_tables: torch.Tensor, ctx_lens: torch.Tensor, out: torch.Tensor,
                     scale: float) -> torch.Tensor:
    _check(qkv, "qkv")
    _check(out, "out")
    if block_tables.dtype != torch.int32 or ctx_lens.dtype != torch.int32:
        raise ValueError("decode_attention: block tables and context lengths must be int32")
    call("ssb_decode_attention", qkv.data_ptr(), qkv.stride(0), nq, nk, pool.data_ptr(),
         _lib.KVGeometry(*geometry), num_blocks, layer, block_tables.data_ptr(), block_tables.shape[1],
         ctx_lens.data_ptr(), ctx_lens.numel(), out.data_ptr(), out.stride(0), scale, _stream())
    return out


def tp_signal_bytes() -> int:
    return int(load().ssb_tp_signal_bytes())


def tp_argmax_keys(key_addrs, sig_addrs, rank: int, rows: int, out_idx: torch.Tensor, epoch: int,
                   max_blocks: int, err: torch.Tensor | None = None) -> None:
    """out_idx[r] = token of the largest LM-head key of row r over every
    rank's keys buffer (peer memory; C-ABI ssb_tp_argmax_keys)."""
    if out_idx.dtype != torch.int32:
        raise ValueError("tp_argmax_keys: out_idx must be int32")
    call("ssb_tp_argmax_keys", _lib.uint64_array(key_addrs), _lib.uint64_array(sig_addrs), len(key_addrs), rank,
         rows, out_idx.data_ptr(), epoch, max_blocks, err.data_ptr() if err is not None else None, _stream())


def lm_head_keys(h: torch.Tensor, w: torch.Tensor, index_base: int, keys: torch.Tensor,
                 workspace: torch.Tensor | None = None, rownorm: "_lib.RowNorm | None" = None) -> None:
    """The LM-head GEMM with its argmax epilogue only: keys[r] = packed
    (logit, index + index_base) maximum of row r (no decode to value/index)."""
    _check(h, "h")
    _check(w, "w")
    M, K = h.shape
    call("ssb_gemm_lm_head_argmax", h.data_ptr(), w.data_ptr(), M, w.shape[0], K, h.stride(0), w.stride(0),
         index_base, keys.data_ptr(), 0, 0, workspace.data_ptr() if workspace is not None else None,
         workspace.numel() * workspace.element_size() if workspace is not None else 0,
         ctypes.byref(rownorm) if rownorm is not None else None, _stream())


def tp_allreduce_rmsnorm(part_addrs, x_addrs, h_addrs, sig_addrs, rank: int, rows: int, hidden: int,
                         gamma: torch.Tensor | None, eps: float, epoch: int, max_blocks: int,
                         err: torch.Tensor | None = None) -> None:
    """x = sum over ranks of part, h = rmsnorm(x) * gamma, written into every
    rank's x / h over NVLink peer memory (C-ABI ssb_tp_allreduce_rmsnorm).
    The address lists are this process's view of every rank's buffers
    (comm.peer_addresses)."""
    n = len(part_addrs)
    if gamma is not None:
        _check(gamma, "gamma")
    call("ssb_tp_allreduce_rmsnorm", _lib.uint64_array(part_addrs), _lib.uint64_array(x_addrs),
         _lib.uint64_array(h_addrs) if h_addrs is not None else None, _lib.uint64_array(sig_addrs), n, rank, rows,
         hidden, hidden, gamma.data_ptr() if gamma is not None else None, eps, epoch, max_blocks,
         err.data_ptr() if err is not None else None, _stream())


def tp_allreduce_rowss(part_addrs, x_addrs, ss_addrs, sig_addrs, rank: int, rows: int, hidden: int, epoch: int,
                       max_blocks: int, err: torch.Tensor | None = None) -> None:
    """x = sum over ranks of part into every rank's x, and the per-row fp32
    sum of squares of x into every rank's ss (the folded-norm combine,
    C-ABI ssb_tp_allreduce_rowss).  Address lists as for
    :func:`tp_allreduce_rmsnorm` (plain lists or prebuilt ctypes arrays)."""
    def arr(a):
        return a if isinstance(a, ctypes.Array) else _lib.uint64_array(a)

    call("ssb_tp_allreduce_rowss", arr(part_addrs), arr(x_addrs), arr(ss_addrs), arr(sig_addrs), len(part_addrs),
         rank, rows, hidden, hidden, epoch, max_blocks, err.data_ptr() if err is not None else None, _stream())


def set_pdl(on: bool) -> bool:
    """Programmatic dependent launch on/off for the library's launches
    (C-ABI ssb_set_pdl); returns the previous setting."""
    return bool(load().ssb_set_pdl(1 if on else 0))
