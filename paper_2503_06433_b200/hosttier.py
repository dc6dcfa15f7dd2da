"""Pinned host KV tier: swap-out under the prefill layout, swap-in under the
decode layout, on a side copy stream ordered by CUDA events.

Reference (/root/reference/pkg/src/shardsim): the CPU tier of
``host_memory_per_gpu * num_gpus`` bytes (specs.py:158-161) buffers prefilled
KV; swap-out overlaps prefill (sim.py:382-385, :417-429); a per-replica FIFO
prefetcher swaps sequences back in while decode runs (sim.py:436-513); the
host layout is HND so head-sharded reads are contiguous (reshard.py:191-201,
PAPER.md:151-154).  Swap-out partitions a sequence by the prefill config's
(layer x head) blocks and swap-in by the decode config's — exactly
``kv_reshard_route`` (reshard.py:170-188): the host tier IS a KV re-shard.

Layout of one sequence's slot: [layer][K|V][head][token][dim] bf16 with
token extent = the prompt length.  A GPU's (layer range x head range) piece is
``2*nl`` rows of ``nh*T*d*2`` bytes at pitch ``H*T*d*2``: one
cudaMemcpy2DAsync each way, staged through a contiguous device buffer filled
/ drained by the ssb_kv_hnd_copy gather / scatter kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .comm import Comm


@dataclass
class SwapTicket:
    seq_id: object
    slot: int
    done: torch.cuda.Event       # recorded on the copy stream when the transfer finished
    staging_idx: int


class HostTier:
    """One replica's shared pinned KV tier plus the copy machinery of one GPU."""

    def __init__(self, comm: Comm, device: torch.device, num_layers: int, num_kv_heads: int, head_dim: int,
                 max_tokens: int, n_slots: int, staging_bytes: int, n_staging: int = 2) -> None:
        self.device = device
        self.L, self.H, self.d = num_layers, num_kv_heads, head_dim
        self.slot_bytes = num_layers * 2 * num_kv_heads * max_tokens * head_dim * 2
        self.n_slots = n_slots
        self.buf = comm.share_host_buffer(self.slot_bytes * n_slots)
        self.free = list(range(n_slots))
        self.copy_stream = torch.cuda.Stream(device)
        self.staging = [torch.empty(max(staging_bytes, 16), dtype=torch.uint8, device=device)
                        for _ in range(n_staging)]
        self.staging_ready: list[torch.cuda.Event | None] = [None] * n_staging
        self._next = 0

    # ------------------------------------------------------------- slots --
    def alloc(self) -> int:
        if not self.free:
            raise RuntimeError("host KV tier has no free slot")
        return self.free.pop(0)

    def release(self, slot: int) -> None:
        self.free.append(slot)
        self.free.sort()

    def _piece(self, slot: int, T: int, gl0: int, nl: int, gh0: int, nh: int) -> tuple[int, int, int, int]:
        """(host address, host pitch, width, height) of a GPU's rectangle."""
        row = self.H * T * self.d * 2
        addr = self.buf.data_ptr() + slot * self.slot_bytes + 2 * gl0 * row + gh0 * T * self.d * 2
        return addr, row, nh * T * self.d * 2, 2 * nl

    def _take_staging(self, stream: torch.cuda.Stream) -> int:
        i = self._next
        self._next = (self._next + 1) % len(self.staging)
        if self.staging_ready[i] is not None:
            stream.wait_event(self.staging_ready[i])
        return i

    # ---------------------------------------------------------- swap-out --
    def swap_out(self, pool: torch.Tensor, geometry, blocks: torch.Tensor, n_tokens: int, slot: int,
                 glayer0: int, ghead0: int, seq_id=None) -> SwapTicket:
        """Gather this GPU's rectangle (current layout) on the compute stream,
        then D2H into the slot on the copy stream."""
        L, H, _, _ = geometry
        compute = torch.cuda.current_stream(self.device)
        i = self._take_staging(compute)
        stg = self.staging[i]
        ops.kv_hnd_copy(True, pool, geometry, blocks, n_tokens, (0, L, 0, H), stg)
        gathered = torch.cuda.Event()
        gathered.record(compute)
        self.copy_stream.wait_event(gathered)
        addr, pitch, width, height = self._piece(slot, n_tokens, glayer0, L, ghead0, H)
        ops.memcpy2d_async(addr, pitch, stg.data_ptr(), width, width, height, stream=self.copy_stream.cuda_stream)
        done = torch.cuda.Event(enable_timing=True)
        done.record(self.copy_stream)
        self.staging_ready[i] = done
        return SwapTicket(seq_id, slot, done, i)

    # ----------------------------------------------------------- swap-in --
    def swap_in(self, pool: torch.Tensor, geometry, blocks: torch.Tensor, n_tokens: int, slot: int,
                glayer0: int, ghead0: int, seq_id=None) -> SwapTicket:
        """H2D of this GPU's rectangle (decode layout) and scatter into the
        pool blocks, both on the copy stream (overlaps decode compute)."""
        L, H, _, _ = geometry
        cs = self.copy_stream
        # the block-id tensor was allocated on the compute stream but is read
        # by the scatter kernel on the copy stream: without this the caching
        # allocator may hand its memory to a compute-stream tensor while the
        # scatter (queued behind hundreds of MB of H2D) has not run yet, and
        # the scatter then writes to garbage block ids (seen at 70B scale)
        blocks.record_stream(cs)
        i = self._take_staging(cs)
        stg = self.staging[i]
        addr, pitch, width, height = self._piece(slot, n_tokens, glayer0, L, ghead0, H)
        ops.memcpy2d_async(stg.data_ptr(), width, addr, pitch, width, height, stream=cs.cuda_stream)
        ops.kv_hnd_copy(False, pool, geometry, blocks, n_tokens, (0, L, 0, H), stg, stream=cs.cuda_stream)
        done = torch.cuda.Event(enable_timing=True)
        done.record(cs)
        self.staging_ready[i] = done
        return SwapTicket(seq_id, slot, done, i)
