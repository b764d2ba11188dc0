"""A/B of compile-time variants of the trailing-update NN GEMM (development tool).

  python tools/nn_variants.py build          # here: one .so per variant under tools/probe/nn_*.so
  python tools/nn_variants.py run [K...]     # on the GPU box: each variant in its own process

Variants are -D macros of csrc/gemm_dmma.cu (QRB_NN_STAGGER_NS, QRB_NN_STAGES);
"head" is the library built from the last commit's sources (/tmp/headsrc/repo)
when present.  Timing: best of 5 CUDA-event runs of C -= V W2, M = 69120,
N = 32768, per K.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tools" / "probe"

VARIANTS = {
    "new": (),
    "stag4k": ("QRB_NN_STAGGER_NS=4000",),
}


def build():
    from paper_1907_01891_b200 import build as b
    for name, defs in VARIANTS.items():
        print(name, b.build(out=OUT / f"nn_{name}.so", defines=defs), flush=True)
    head = Path("/tmp/headsrc/repo")
    if head.is_dir():
        r = subprocess.run([sys.executable, "-c",
                            "import sys; sys.path.insert(0, '.'); "
                            "from paper_1907_01891_b200 import build as b; "
                            f"print(b.build(out=__import__('pathlib').Path('{OUT}/nn_head.so')))"],
                           cwd=head, capture_output=True, text=True)
        print("head", r.stdout.strip(), r.stderr[-500:])


def run_one(ks):
    import ctypes

    import torch
    from paper_1907_01891_b200 import _native
    lib = _native.load()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    M, N = 69120, 32768
    res = {}
    for K in ks:
        V = torch.randn(K, M, dtype=torch.float64, device="cuda")
        W = torch.randn(N, K, dtype=torch.float64, device="cuda")
        C = torch.randn(N, M, dtype=torch.float64, device="cuda")
        f = lambda: lib.qrb_op_gemm_nn_sub(P(V), M, P(W), K, P(C), M, M, N, K, None)  # noqa
        f()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        res[K] = round(2 * M * N * K / best / 1e9, 3)
        # the W = V^T C product of the same step (TN, one 128 x 64 tile over all M per CTA)
        Wt = torch.zeros(N, K, dtype=torch.float64, device="cuda")
        g = lambda: lib.qrb_op_gemm_tn(P(V), M, P(C), M, P(Wt), K, K, N, M, 1, 0, 0, None)  # noqa
        g()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        res[f"tn{K}"] = round(2 * M * N * K / best / 1e9, 3)
        del V, W, C, Wt
    return res


def run(ks):
    out = {}
    for so in sorted(OUT.glob("nn_*.so")):
        env = dict(os.environ, QRB_LIB_PATH=str(so))
        r = subprocess.run([sys.executable, __file__, "one", *map(str, ks)], env=env,
                           capture_output=True, text=True, timeout=600)
        try:
            out[so.stem] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            out[so.stem] = r.stderr[-400:]
        print(so.stem, out[so.stem], flush=True)
    return out


if __name__ == "__main__":
    cmd = sys.argv[1]
    ks = [int(x) for x in sys.argv[2:]] or [256, 512]
    if cmd == "build":
        build()
    elif cmd == "one":
        print(json.dumps(run_one(ks)))
    else:
        run(ks)
