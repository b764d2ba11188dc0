"""qrb_factorize_host_gated: the factorization copies a column chunk only once
its ready flag is up (the drop-in factorize's tile readers fill the host matrix
while the GPU already works), reports how many leading columns are final, and
returns an error instead of waiting forever when a chunk is marked unreadable.
Same chunk schedule as qrb_factorize_host -> the same bits."""

import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _problem(m=3000, n=2176, seed=3):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (u * np.linspace(30, 1, n)) @ v.T


def test_gated_factorization_equals_ungated_and_reports_progress():
    from paper_1907_01891_b200.device import PinnedHostArray, QrDevice
    a = _problem()
    m, n = a.shape
    lda = (m + 31) // 32 * 32
    chunk = 512
    nchunks = -(-n // chunk)
    host = PinnedHostArray((n, lda))
    ready = PinnedHostArray((nchunks,), np.int32)
    prog = PinnedHostArray((1,), np.int64)
    view = host.array.T
    ready.array[:] = 0
    prog.array[0] = 0
    seen = []

    def fill():                                   # a slow "reader": one chunk per 20 ms
        for c in range(nchunks):
            c0, c1 = c * chunk, min(n, (c + 1) * chunk)
            view[:m, c0:c1] = a[:, c0:c1]
            ready.array[c] = 1
            seen.append(int(prog.array[0]))
            time.sleep(0.02)

    th = threading.Thread(target=fill)
    with QrDevice(m, n) as q:
        th.start()
        q.factorize_host_gated(view[:m], chunk, ready.array, input_gbps=45.0,
                               progress=prog.array)
        th.join()
        gated = q.get_matrix()
        assert int(prog.array[0]) == n
        assert seen == sorted(seen) and seen[-1] < n     # progress grows while chunks arrive
        q.factorize_host(np.asfortranarray(a), chunk_cols=chunk)
        np.testing.assert_array_equal(q.get_matrix(), gated)
    for h in (host, ready, prog):
        h.close()


def test_gated_factorization_aborts_on_an_unreadable_chunk():
    from paper_1907_01891_b200.device import PinnedHostArray, QrDevice
    from paper_1907_01891_b200.errors import GpuError
    a = _problem(1200, 900, 4)
    m, n = a.shape
    lda = (m + 31) // 32 * 32
    host = PinnedHostArray((n, lda))
    ready = PinnedHostArray((2,), np.int32)
    host.array.T[:m] = a
    ready.array[:] = [1, -1]
    with QrDevice(m, n) as q:
        with pytest.raises(GpuError, match="unavailable"):
            q.factorize_host_gated(host.array.T[:m], 512, ready.array)
    host.close()
    ready.close()
