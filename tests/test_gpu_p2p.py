"""Point-to-point send / recv / sendrecv on the device mailboxes (emulated
ranks on cuda:0), with the reference transport's contract
(transport/base.py:140-152, tests/test_transport_inprocess.py): exact
(source, tag) FIFO matching, sends that never wait for the receiver, empty
payloads, SelfSend / LengthMismatch / tag checks, plus messages larger than a
mailbox ring (fragments) exchanged symmetrically without deadlock."""
import threading
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2504_18658_b200 as pkg

    return pkg


def test_loopback_round_trip():
    pkg = _pkg()
    payload = np.arange(16, dtype=np.float32).tobytes()

    def fn(c):
        if c.rank == 0:
            c.send(1, 7, payload)
            return None
        return c.recv(0, 7)

    assert pkg.run_ranks(2, fn)[1] == payload


def test_fifo_per_channel_and_tag_matching_out_of_order():
    pkg = _pkg()

    def fn(c):
        if c.rank == 0:
            c.send(1, 3, b"AAAA")
            c.send(1, 4, b"CCCC")
            c.send(1, 3, b"BBBB")
            return None
        return c.recv(0, 4), c.recv(0, 3), c.recv(0, 3)

    assert pkg.run_ranks(2, fn)[1] == (b"CCCC", b"AAAA", b"BBBB")


def test_contract_errors():
    pkg = _pkg()
    E = pkg.errors
    with pytest.raises(E.SelfSend):
        pkg.run_ranks(2, lambda c: c.send(c.rank, 0, b""))
    with pytest.raises(E.LengthMismatch):
        pkg.run_ranks(2, lambda c: c.send(1, 0, b"abc") if c.rank == 0 else None)
    with pytest.raises(ValueError):
        pkg.run_ranks(2, lambda c: c.send(1, -1, b"") if c.rank == 0 else None)
    with pytest.raises(E.SelfSend):
        pkg.run_ranks(1, lambda c: c.sendrecv(0, 0, b""))


def test_recv_posted_before_send():
    pkg = _pkg()

    def fn(c):
        if c.rank == 1:
            return c.recv(0, 5)
        time.sleep(0.05)
        c.send(1, 5, b"late")
        return None

    assert pkg.run_ranks(2, fn)[1] == b"late"


def test_sendrecv_exchange_empty_and_disjoint_pairs():
    pkg = _pkg()
    res = pkg.run_ranks(2, lambda c: c.sendrecv(1 - c.rank, 9, bytes([c.rank + 1] * 4)))
    assert res == [bytes([2] * 4), bytes([1] * 4)]
    assert pkg.run_ranks(2, lambda c: c.sendrecv(1 - c.rank, 2, b"")) == [b"", b""]
    res = pkg.run_ranks(4, lambda c: c.sendrecv(c.rank ^ 1, 4, bytes([c.rank] * 4)))
    assert res == [bytes([r ^ 1] * 4) for r in range(4)]


@pytest.mark.parametrize("nbytes", [4, 1 << 20, (5 << 20) + 12])
def test_large_symmetric_exchange_fragments_without_deadlock(nbytes):
    """Both ranks send first (messages larger than a 2 MiB ring): each drains
    its own rings while waiting for space, so both sends complete."""
    pkg = _pkg()
    rng = np.random.default_rng(nbytes)
    msgs = [rng.integers(0, 256, nbytes, dtype=np.uint8).tobytes() for _ in range(2)]
    res = pkg.run_ranks(2, lambda c: c.sendrecv(1 - c.rank, 11, msgs[c.rank]))
    assert res[0] == msgs[1] and res[1] == msgs[0]


def test_device_tensors_and_many_messages():
    pkg = _pkg()
    p = 4

    def fn(c):
        out = []
        for it in range(50):  # ring wrap-around many times
            for d in range(p):
                if d != c.rank:
                    c.send(d, it, torch.full((1000,), float(c.rank * 100 + it), device="cuda"))
            got = {}
            for s in range(p):
                if s != c.rank:
                    t = torch.empty(1000, device="cuda")
                    c.recv_into(s, it, t)
                    got[s] = float(t[0]) if bool((t == t[0]).all()) else None
            out.append(got)
        return out

    res = pkg.run_ranks(p, fn)
    for r in range(p):
        for it, got in enumerate(res[r]):
            assert got == {s: float(s * 100 + it) for s in range(p) if s != r}


def test_recv_times_out_instead_of_hanging():
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(2, 0)
    w.set_timeout_ms(300)
    try:
        with pytest.raises(pkg.errors.Timeout):
            pkg.run_ranks(2, lambda c: c.recv(1 - c.rank, 99))
    finally:
        w.set_timeout_ms(20000)
