"""CPU oracle for the hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package's tiled out-of-core QR and solve
(``oocqr``: kernels.py, task_engine.py), used only as the parity checker by
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py``.  Nothing in the product package
imports it; the product path fails loudly when the CUDA library is missing.

Parity of this restatement is pinned against the reference itself: the golden
fixtures under ``tests/golden/`` were produced by running the reference
(``/root/reference/pkg/src``) in this container with the committed script
``tests/golden/make_golden.py``; ``tests/test_oracle.py`` checks the oracle
against every one of them.
"""

from .tiled_qr import (  # noqa: F401
    OracleFactors,
    apply_left_qt_dense,
    apply_left_qt_td,
    comp_dense_qr,
    comp_td_qr,
    factorize_dense,
    gemm_nn_mo,
    gen_factorization_tasks,
    gen_solve_tasks,
    solve_dense,
    trsm_lunn,
)
