"""comm._IpcMapping: one cudaIpcOpenMemHandle per (allocation handle, device)
in a process, shared by every peer buffer carved from that allocation, and
closed with its last holder (TorchComm.peer_addresses).  The library calls
are replaced by a recording fake, so this runs without a GPU."""

from __future__ import annotations

import gc

import pytest

from paper_2503_06433_b200 import _lib, comm


class _FakeLib:
    def __init__(self) -> None:
        self.opened: list = []
        self.closed: list = []
        self.next_ptr = 0x7000_0000

    def ssb_ipc_open(self, handle, device, out) -> int:
        self.opened.append((bytes(handle), device))
        out._obj.value = self.next_ptr
        self.next_ptr += 0x1000_0000
        return 0

    def ssb_ipc_close(self, ptr, device) -> int:
        self.closed.append((ptr, device))
        return 0

    def ssb_last_error(self) -> bytes:
        return b""


@pytest.fixture
def fake(monkeypatch):
    lib = _FakeLib()
    monkeypatch.setattr(_lib, "load", lambda: lib)
    comm._IpcMapping._open.clear()
    yield lib
    comm._IpcMapping._open.clear()


def test_one_open_per_allocation_and_close_with_last_holder(fake):
    h = b"\x01" * 64
    a = comm._IpcMapping.open(h, 0)
    b = comm._IpcMapping.open(h, 0)  # another buffer of the same allocation
    assert a.base == b.base and len(fake.opened) == 1
    del a
    gc.collect()
    assert fake.closed == []
    del b
    gc.collect()
    assert fake.closed == [(0x7000_0000, 0)]
    c = comm._IpcMapping.open(h, 0)  # reopened after the last close
    assert len(fake.opened) == 2 and c.base != 0x7000_0000


def test_distinct_handles_and_devices_map_separately(fake):
    x = comm._IpcMapping.open(b"\x02" * 64, 0)
    y = comm._IpcMapping.open(b"\x03" * 64, 0)
    z = comm._IpcMapping.open(b"\x02" * 64, 1)
    assert len({x.base, y.base, z.base}) == 3 and len(fake.opened) == 3
    del x, y, z
    gc.collect()
    assert len(fake.closed) == 3


def test_open_failure_raises(fake, monkeypatch):
    monkeypatch.setattr(fake, "ssb_ipc_open", lambda h, d, out: -1)
    with pytest.raises(_lib.SeesawKernelError):
        comm._IpcMapping.open(b"\x04" * 64, 0)
    assert comm._IpcMapping._open == {}
