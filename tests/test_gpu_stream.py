"""qrb_factorize_host: chunked host->HBM copy overlapped with a left-looking
chunk order -- same factors as the right-looking in-HBM factorization."""

import numpy as np
import pytest

from conftest import rel_err, sign_normalise
from oracle import tiled_qr as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,nb,chunk", [(3000, 1100, 128, 256), (2000, 2000, 64, 640),
                                          (1500, 700, 32, 0), (4100, 1300, 128, 1300)])
def test_factorize_host_matches_in_hbm(m, n, nb, chunk):
    import torch

    from paper_1907_01891_b200.device import QrDevice

    rng = np.random.default_rng(m + n + nb)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.linspace(30, 1, n)) @ v.T
    lda = (m + 31) // 32 * 32
    pin = torch.zeros((n, lda), dtype=torch.float64, pin_memory=True)
    pin[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    view = pin.numpy().T[:m, :]
    bm = rng.standard_normal((m, 4))
    with QrDevice(m, n, nb) as q:
        rep = q.factorize_host(view, chunk_cols=chunk)
        assert rep["h2d_bytes"] == 8 * m * n and rep["flops"] > 0
        r_s = q.r_factor()
        x_s, res_s, _ = q.solve(bm)
        q.set_matrix(a)
        q.factorize()
        r_h = q.r_factor()
        x_h, res_h, _ = q.solve(bm)
    assert rel_err(r_s, r_h) <= 1e-12          # same dlarfg signs, different summation order
    assert rel_err(x_s, x_h) <= 1e-10
    f = orc.factorize_dense(a, 256, 64)
    assert rel_err(sign_normalise(r_s), sign_normalise(f.r())) <= 1e-10
    assert rel_err(x_s, orc.solve_dense(f, bm)) <= 1e-8
    np.testing.assert_allclose(res_s, res_h, rtol=1e-9)


def test_factorize_host_rejects_non_finite():
    import paper_1907_01891_b200 as pkg
    from paper_1907_01891_b200.device import QrDevice

    a = np.random.default_rng(1).standard_normal((900, 400))
    a[123, 301] = np.nan
    with QrDevice(900, 400) as q:
        with pytest.raises(pkg.KernelInputError):
            q.factorize_host(a, chunk_cols=128)


def test_two_handles_on_two_streams_from_two_threads():
    """The per-device workspace shared by every handle (qrb_api.cu WsUse): two
    handles on different streams, factored and solved concurrently from two
    host threads, give exactly the results of running them one after the
    other."""
    import threading

    import numpy as np
    import torch
    from paper_1907_01891_b200.device import QrDevice

    rng = np.random.default_rng(17)
    mats = [rng.standard_normal((2600, 1300)), rng.standard_normal((3100, 1700))]
    rhs = [rng.standard_normal((a.shape[0], 4)) for a in mats]

    def run(i, out, stream=None):
        with QrDevice(*mats[i].shape) as q:
            if stream is not None:
                q.set_stream(stream.cuda_stream)
            q.set_matrix(mats[i])
            q.factorize()
            x, _, _ = q.solve(rhs[i])
            out[i] = (q.get_matrix(), x)

    ref = {}
    for i in range(2):
        run(i, ref)
    got = {}
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ths = [threading.Thread(target=run, args=(i, got, streams[i])) for i in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i in range(2):
        np.testing.assert_array_equal(got[i][0], ref[i][0])
        np.testing.assert_array_equal(got[i][1], ref[i][1])
