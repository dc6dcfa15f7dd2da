"""Collective plumbing for the SPMD workers (one process — or thread — per GPU).

The engine only needs five operations over a *group* of ranks: all-to-all
with uneven splits (weight and KV re-shard), in-place sum all-reduce (TP
row-parallel outputs), all-gather (vocab-parallel argmax), point-to-point
send/recv (PP activations) and barrier.

* :class:`TorchComm` — ``torch.distributed`` groups: NCCL over NVLink/NVSwitch
  on the GPU box (one process per GPU, launched by torchrun), gloo on CPU for
  the multi-process tests.  NCCL is reached only through torch so exactly one
  libnccl (torch's bundled 2.28) lives in the process.
* :class:`ThreadComm` — W virtual ranks as threads of one process sharing one
  device.  Used to run and test the multi-rank PP→TP path bit-exactly on a
  single GPU (the only configuration gpurun provides); transfers are device
  copies between the ranks' buffers, ordered by stream synchronisation.
"""

from __future__ import annotations

import threading
from typing import Sequence

import torch


class Comm:
    """Interface: a group of ``size`` ranks; ``rank`` is this member's index."""

    rank: int
    size: int

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits: Sequence[int],
                   in_splits: Sequence[int]) -> None:
        raise NotImplementedError

    def all_reduce_(self, t: torch.Tensor) -> None:
        raise NotImplementedError

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        """out = concat over ranks (dim 0) of inp."""
        raise NotImplementedError

    def send(self, t: torch.Tensor, dst: int) -> None:
        raise NotImplementedError

    def recv(self, t: torch.Tensor, src: int) -> None:
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError

    def subgroup(self, members: Sequence[int]) -> "Comm":
        """Group of the listed ranks (indices in THIS group); every member of
        this group must call it with the same lists in the same order."""
        raise NotImplementedError

    def share_host_buffer(self, nbytes: int) -> torch.Tensor:
        """A pinned host buffer visible to every member of the group (the
        shared host KV tier).  Collective."""
        raise NotImplementedError

    def peer_addresses(self, t: torch.Tensor, keep: list) -> list[int]:
        """Device addresses, valid in THIS process, of every member's ``t``
        (the tensor each member passes): the local pointer for self, CUDA IPC
        mappings (NVLink peer memory) for the others.  The objects that keep
        the mappings open are appended to ``keep``: the caller owns them (the
        buffer's owner), so a mapping closes when its owner is released.
        Collective."""
        raise NotImplementedError


def _pinned(nbytes: int) -> torch.Tensor:
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=torch.cuda.is_available())


class SoloComm(Comm):
    """A group of one."""

    def __init__(self) -> None:
        self.rank, self.size = 0, 1

    def all_to_all(self, out, inp, out_splits, in_splits) -> None:
        if out.data_ptr() != inp.data_ptr():
            out[: int(in_splits[0])].copy_(inp[: int(in_splits[0])])

    def all_reduce_(self, t) -> None:
        return None

    def all_gather(self, out, inp) -> None:
        out.view(-1)[: inp.numel()].copy_(inp.reshape(-1))

    def send(self, t, dst) -> None:
        raise RuntimeError("send in a group of one")

    def recv(self, t, src) -> None:
        raise RuntimeError("recv in a group of one")

    def barrier(self) -> None:
        return None

    def subgroup(self, members) -> Comm:
        return self

    def share_host_buffer(self, nbytes: int) -> torch.Tensor:
        return _pinned(nbytes)

    def peer_addresses(self, t: torch.Tensor, keep: list) -> list[int]:
        return [t.data_ptr()]


class TorchComm(Comm):
    """torch.distributed process group: NCCL on the GPU boxes (one process
    per GPU).  With the gloo backend, CUDA tensors are staged through host
    memory — the path the multi-process tests use to run the real SPMD engine
    as several processes on the single GPU a test box has; it is never the
    data path of a multi-GPU run."""

    def __init__(self, group=None, ranks: Sequence[int] | None = None) -> None:
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.global_ranks = list(ranks) if ranks is not None else list(range(dist.get_world_size()))
        self.size = len(self.global_ranks)
        self.rank = self.global_ranks.index(dist.get_rank())
        self._host_staged = dist.get_backend(group) == "gloo"

    def _stage(self, t: torch.Tensor) -> torch.Tensor:
        if self._host_staged and t.is_cuda:
            return t.detach().cpu()
        return t

    @staticmethod
    def _unstage(dst: torch.Tensor, host: torch.Tensor) -> None:
        if host.data_ptr() != dst.data_ptr():
            dst.copy_(host)

    def all_to_all(self, out, inp, out_splits, in_splits) -> None:
        os_, is_ = [int(x) for x in out_splits], [int(x) for x in in_splits]
        # staging buffers are allocated for the largest chunk: pass exact views
        o, i = out[: sum(os_)], inp[: sum(is_)]
        ho, hi = self._stage(o), self._stage(i)
        self._dist.all_to_all_single(ho, hi, os_, is_, group=self.group)
        self._unstage(o, ho)

    def all_reduce_(self, t) -> None:
        if self.size > 1:
            h = self._stage(t)
            self._dist.all_reduce(h, group=self.group)
            self._unstage(t, h)

    def all_gather(self, out, inp) -> None:
        ho = self._stage(out)
        self._dist.all_gather_into_tensor(ho, self._stage(inp.contiguous()), group=self.group)
        self._unstage(out, ho)

    def send(self, t, dst) -> None:
        self._dist.send(self._stage(t), self.global_ranks[dst], group=self.group)

    def recv(self, t, src) -> None:
        h = self._stage(t)
        self._dist.recv(h, self.global_ranks[src], group=self.group)
        self._unstage(t, h)

    def barrier(self) -> None:
        if self.size > 1:
            self._dist.barrier(group=self.group)

    def subgroup(self, members) -> Comm:
        ranks = [self.global_ranks[m] for m in members]
        if len(ranks) == 1:
            solo = SoloComm()
            return solo
        # new_group must be entered by every process of the default group
        group = _new_group_cached(self._dist, tuple(ranks))
        return TorchComm(group, ranks) if self._dist.get_rank() in ranks else SoloComm()

    def share_host_buffer(self, nbytes: int) -> torch.Tensor:
        """POSIX shared memory created by the group's first rank, mapped and
        cudaHostRegister'ed by every process: one host KV tier per replica
        without the two-stage GPU->pinned->shared copy of PAPER.md:133."""
        from multiprocessing import shared_memory

        name = [None]
        if self.rank == 0:
            shm = shared_memory.SharedMemory(create=True, size=max(nbytes, 1))
            name = [shm.name]
        self._dist.broadcast_object_list(name, src=self.global_ranks[0], group=self.group)
        if self.rank != 0:
            shm = shared_memory.SharedMemory(name=name[0])
        buf = torch.frombuffer(shm.buf, dtype=torch.uint8, count=max(nbytes, 1))
        if torch.cuda.is_available():
            rc = torch.cuda.cudart().cudaHostRegister(buf.data_ptr(), buf.numel(), 1)  # portable
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister of the shared host tier failed ({rc})")
        _SHM_KEEPALIVE.append(shm)
        self.barrier()
        return buf


    def peer_addresses(self, t: torch.Tensor, keep: list) -> list[int]:
        """CUDA IPC: every member exports the cudaMalloc allocation holding
        ``t`` (handle + offset, ssb_ipc_export), the others map it in the
        context of THEIR OWN device (ssb_ipc_open, peer access enabled on
        open), so their kernels can dereference it over NVLink.  (torch's
        shared-storage path would map it under the exporter's device index:
        a context on the peer GPU, and no peer access for the local one.)
        The mappings go to ``keep``; each is closed when the last holder of
        its allocation drops it."""
        import ctypes

        from . import _lib

        lib = _lib.load()
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_int64(0)
        rc = lib.ssb_ipc_export(ctypes.c_void_p(t.data_ptr()), handle, ctypes.byref(off))
        if rc != 0:
            raise _lib.SeesawKernelError(f"ssb_ipc_export failed ({rc}): {lib.ssb_last_error().decode()}")
        mine = (bytes(handle.raw), int(off.value))
        objs: list = [None] * self.size
        self._dist.all_gather_object(objs, mine, group=self.group)
        dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
        addrs = []
        for r, (h, o) in enumerate(objs):
            if r == self.rank:
                addrs.append(t.data_ptr())
                continue
            m = _IpcMapping.open(h, dev)
            keep.append(m)
            addrs.append(m.base + o)
        return addrs


class _IpcMapping:
    """A peer allocation mapped into this process (one cudaIpcOpenMemHandle
    per (handle, device), shared by every buffer carved from it; closed with
    its last holder)."""

    _open: dict = {}
    _lock = threading.RLock()  # re-entrant: a GC-triggered __del__ may run inside open()

    def __init__(self, key, base: int) -> None:
        self.key, self.base = key, base

    @classmethod
    def open(cls, handle: bytes, device: int) -> "_IpcMapping":
        import ctypes

        from . import _lib

        key = (handle, device)
        with cls._lock:
            ent = cls._open.get(key)
            if ent is None:
                lib = _lib.load()
                ptr = ctypes.c_void_p(0)
                rc = lib.ssb_ipc_open(handle, device, ctypes.byref(ptr))
                if rc != 0:
                    raise _lib.SeesawKernelError(f"ssb_ipc_open failed ({rc}): {lib.ssb_last_error().decode()}")
                ent = cls._open[key] = [int(ptr.value), 0]
            ent[1] += 1
            return cls(key, ent[0])

    def __del__(self) -> None:
        try:
            with self._lock:
                ent = self._open.get(self.key)
                if ent is None:
                    return
                ent[1] -= 1
                if ent[1] == 0:
                    del self._open[self.key]
                    from . import _lib

                    _lib.load().ssb_ipc_close(ent[0], self.key[1])
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_GROUPS: dict[tuple[int, ...], object] = {}
_SHM_KEEPALIVE: list = []


def _new_group_cached(dist, ranks: tuple[int, ...]):
    if ranks not in _GROUPS:
        _GROUPS[ranks] = dist.new_group(list(ranks))
    return _GROUPS[ranks]


class _ThreadWorld:
    """Shared state of W thread-ranks.  Every wait is bounded (TIMEOUT_S):
    a rank that died leaves the others with BrokenBarrierError / TimeoutError
    instead of a hang."""

    TIMEOUT_S = 300.0

    def __init__(self, size: int) -> None:
        self.size = size
        self.barrier = threading.Barrier(size, timeout=self.TIMEOUT_S)
        self.slots: dict = {}
        self.lock = threading.Lock()
        self.mail: dict[tuple[int, int, int], torch.Tensor] = {}
        self.mail_cv = threading.Condition()
        self.subworlds: dict[tuple[int, ...], "_ThreadWorld"] = {}


class ThreadComm(Comm):
    """Virtual ranks = threads of one process on one device."""

    def __init__(self, world: _ThreadWorld, rank: int) -> None:
        self.world = world
        self.rank = rank
        self.size = world.size
        self._seq: dict[tuple[int, int], int] = {}

    @staticmethod
    def create(size: int) -> list["ThreadComm"]:
        w = _ThreadWorld(size)
        return [ThreadComm(w, r) for r in range(size)]

    def _sync(self) -> None:
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()

    def _exchange(self, obj):
        """Publish ``obj`` and return everyone's published objects."""
        self._sync()
        w = self.world
        with w.lock:
            w.slots[self.rank] = obj
        w.barrier.wait()
        objs = [w.slots[r] for r in range(self.size)]
        return objs

    def _done(self) -> None:
        self._sync()
        self.world.barrier.wait()

    def all_to_all(self, out, inp, out_splits, in_splits) -> None:
        objs = self._exchange((inp, [int(x) for x in in_splits]))
        src_offs = []
        for tensor, splits in objs:
            offs, acc = [], 0
            for s in splits:
                offs.append(acc)
                acc += s
            src_offs.append(offs)
        pos = 0
        for q in range(self.size):
            n = int(out_splits[q])
            tensor, splits = objs[q]
            if splits[self.rank] != n:
                raise RuntimeError(f"all_to_all split mismatch {splits[self.rank]} != {n}")
            if n:
                o = src_offs[q][self.rank]
                out[pos : pos + n].copy_(tensor[o : o + n])
            pos += n
        self._done()

    def all_reduce_(self, t) -> None:
        if self.size == 1:
            return
        objs = self._exchange(t)
        acc = objs[0].float().clone()
        for x in objs[1:]:
            acc += x.float()
        self._sync()
        self.world.barrier.wait()  # everyone has read the inputs
        t.copy_(acc.to(t.dtype))
        self._done()

    def all_gather(self, out, inp) -> None:
        objs = self._exchange(inp)
        n = inp.numel()
        flat = out.view(-1)
        for q, x in enumerate(objs):
            flat[q * n : (q + 1) * n].copy_(x.reshape(-1))
        self._done()

    def _key(self, src: int, dst: int) -> tuple[int, int, int]:
        k = (src, dst)
        self._seq[k] = self._seq.get(k, 0) + 1
        return (src, dst, self._seq[k])

    def send(self, t, dst) -> None:
        self._sync()
        key = self._key(self.rank, dst)
        w = self.world
        with w.mail_cv:
            w.mail[key] = t
            w.mail_cv.notify_all()
            # rendezvous: wait until the receiver consumed it (buffer reuse safety)
            if not w.mail_cv.wait_for(lambda: key not in w.mail, timeout=w.TIMEOUT_S):
                raise TimeoutError(f"ThreadComm send {key}: receiver never took it")

    def recv(self, t, src) -> None:
        key = self._key(src, self.rank)
        w = self.world
        with w.mail_cv:
            if not w.mail_cv.wait_for(lambda: key in w.mail, timeout=w.TIMEOUT_S):
                raise TimeoutError(f"ThreadComm recv {key}: sender never posted it")
            t.copy_(w.mail[key])
            self._sync()
            del w.mail[key]
            w.mail_cv.notify_all()

    def barrier(self) -> None:
        self._done()

    def share_host_buffer(self, nbytes: int) -> torch.Tensor:
        objs = self._exchange(_pinned(nbytes) if self.rank == 0 else None)
        buf = objs[0]
        self._done()
        return buf

    def peer_addresses(self, t: torch.Tensor, keep: list) -> list[int]:
        objs = self._exchange(t.data_ptr())
        self._done()
        return list(objs)

    def subgroup(self, members) -> Comm:
        members = tuple(members)
        if len(members) == 1:
            return SoloComm()
        w = self.world
        with w.lock:
            if members not in w.subworlds:
                w.subworlds[members] = _ThreadWorld(len(members))
            sub = w.subworlds[members]
        if self.rank not in members:
            return SoloComm()
        return ThreadComm(sub, members.index(self.rank))
