"""The NVLink peer-memory one-shot allreduce (peer.cu, SDR_PEER=1 on several
ranks), emulated as one kernel over all ranks' data: every virtual rank is a
CTA of one cooperative launch on this GPU with its own symmetric buffer, the
peers' buffers reached through plain device pointers. Several epochs back to
back exercise the parity double-buffering and the epoch flags; every rank
must hold exactly the rank-ordered sum."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,n,epochs", [(2, 5, 3), (4, 490, 6), (8, 1024, 5), (8, 1, 9), (3, 257, 4)])
def test_peer_allreduce_emulated(sk, world, n, epochs):
    rng = np.random.default_rng(world * 1000 + n)
    vals = rng.standard_normal((epochs, world, n))
    out = np.zeros_like(vals)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    sk._check(sk._lib.sdr_debug_peer_emulate(world, n, epochs, p(vals), p(out)))
    for e in range(epochs):
        ref = np.zeros(n)
        for q in range(world):  # the kernel's order: rank 0, 1, ...
            ref = ref + vals[e, q]
        for r in range(world):
            assert np.array_equal(out[e, r], ref), (e, r)


def test_peer_allreduce_rejects_oversize(sk):
    v = np.zeros(2 * 2000)
    o = np.zeros_like(v)
    with pytest.raises(ValueError):
        sk._check(sk._lib.sdr_debug_peer_emulate(2, 2000, 1, v.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p)))
