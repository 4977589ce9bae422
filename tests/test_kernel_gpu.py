"""K1 tile kernel (tcgen05/TMEM/TMA) vs a float64 torch reference.

Replaces the reference's per-tile numpy kernel (tiles.py:154-179); numerics
are checked with the north-star tolerances (relative Frobenius error <= 1e-5
for the FP32-accurate split-bf16 mode, <= 1e-2 for bf16) on zero-mean normal
inputs, and bit-exactly on small-integer inputs (exact in bf16 and fp32).
"""

import pytest
import torch

from paper_1511_04348_b200 import dense_gemm
from paper_1511_04348_b200.dense import set_gemm_pairs

pytestmark = pytest.mark.gpu

TOL = {"fp32acc": 1e-5, "bf16": 1e-2, "fp32hi": 2e-6}


def rel_fro(c, ref):
    return float(torch.linalg.norm(c.double() - ref) / torch.linalg.norm(ref))


def make(m, k, n, ta, tb, dtype, gen, kind="normal"):
    def mk(r, c):
        if kind == "int":
            return torch.randint(-4, 5, (r, c), generator=gen, dtype=torch.int64).to(dtype)
        return torch.randn((r, c), generator=gen, dtype=torch.float64).to(dtype)

    a = mk(k, m) if ta else mk(m, k)
    b = mk(n, k) if tb else mk(k, n)
    return a.cuda(), b.cuda()


def ref_product(a, b, ta, tb):
    a64, b64 = a.double(), b.double()
    return (a64.T if ta else a64) @ (b64.T if tb else b64)


SHAPES = [(128, 256, 64), (1, 1, 1), (5, 7, 3), (200, 300, 130), (257, 513, 1000), (1024, 768, 4096)]


@pytest.fixture(params=[False, True], ids=["cta", "cta_pair"])
def variant(request):
    set_gemm_pairs(request.param)
    yield request.param
    set_gemm_pairs(False)


@pytest.mark.parametrize("precision", ["fp32acc", "bf16", "fp32hi"])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("shape", SHAPES)
def test_dense_kernel_normal(shape, ta, tb, precision, variant):
    m, n, k = shape
    gen = torch.Generator().manual_seed(hash((shape, ta, tb)) & 0xFFFF)
    a, b = make(m, k, n, ta, tb, torch.float32, gen)
    c = dense_gemm(a, b, ta, tb, precision=precision)
    torch.cuda.synchronize()
    err = rel_fro(c, ref_product(a, b, ta, tb))
    assert err <= TOL[precision], f"{shape} ta={ta} tb={tb} {precision}: rel err {err:.3e}"


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_dense_kernel_integers_exact(ta, tb, variant):
    gen = torch.Generator().manual_seed(7)
    for (m, n, k) in [(33, 65, 17), (300, 260, 700)]:
        a, b = make(m, k, n, ta, tb, torch.float64, gen, kind="int")
        for precision in ("bf16", "fp32acc", "fp32hi"):
            c = dense_gemm(a, b, ta, tb, precision=precision)
            torch.cuda.synchronize()
            assert torch.equal(c, ref_product(a, b, ta, tb)), precision


def test_dense_kernel_accumulate_and_f64_out(variant):
    gen = torch.Generator().manual_seed(3)
    a, b = make(130, 70, 300, False, False, torch.float64, gen)
    c0 = torch.randn((130, 300), dtype=torch.float64, generator=gen).cuda()
    c = c0.clone()
    dense_gemm(a, b, out=c, accumulate=True)
    torch.cuda.synchronize()
    ref = c0 + ref_product(a, b, False, False)
    assert rel_fro(c, ref) <= 1e-5


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
def test_tma_multicast_clusters_match(precision):
    """The opt-in TMA-multicast K1 (clusters of two CTA pairs sharing their A
    tile, tr_set_gemm_multicast) against the float64 oracle and against the
    default CTA-pair kernel, on a grouped warm product with ragged rows."""
    import numpy as np

    from paper_1511_04348_b200 import Runtime, homogeneous_machine
    from paper_1511_04348_b200 import _native as N

    T = 1024
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(3 * T + 300, 2 * T + 64, device="cuda", generator=g)
    b = torch.randn(2 * T + 64, 4 * T, device="cuda", generator=g)
    outs = {}
    for mc in (0, 1):
        N.call("tr_set_gemm_multicast", mc)
        try:
            c = torch.empty(a.shape[0], b.shape[1], device="cuda")
            with Runtime(homogeneous_machine(1, dtype=np.float32), T, precision=precision) as rt:
                for _ in range(2):  # the second product is warm: grouped persistent launches
                    rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
            outs[mc] = c.double()
        finally:
            N.call("tr_set_gemm_multicast", 0)
    ref = a.double() @ b.double()
    tol = 1e-5 if precision == "fp32acc" else 1e-2
    for mc in (0, 1):
        assert float(torch.linalg.norm(outs[mc] - ref) / torch.linalg.norm(ref)) <= tol
    # every output element goes through the same MMA sequence either way
    assert torch.equal(outs[0], outs[1])


def test_die_aware_unit_order_is_measured_and_bitwise_neutral(tmp_path):
    """K1's die map (L2 latency signatures of every SM + the pair grid's
    placement) splits the 74 pair clusters between the two dies, and the
    die-aware unit order changes only which cluster computes which tile: the
    grouped warm product is bit-identical with it off (TR_K1_DIE=0)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    import numpy as np

    from paper_1511_04348_b200.dense import k1_die_map

    n0, n1 = k1_die_map(0)
    assert n0 + n1 == torch.cuda.get_device_properties(0).multi_processor_count // 2
    assert min(n0, n1) >= (n0 + n1) // 4
    code = (
        "import sys, numpy as np, torch\n"
        "import paper_1511_04348_b200 as tr\n"
        "g = torch.Generator(device='cuda').manual_seed(5)\n"
        "A = torch.randn(8192, 4096, device='cuda', generator=g)\n"
        "B = torch.randn(4096, 8192, device='cuda', generator=g)\n"
        "C = torch.empty(8192, 8192, device='cuda')\n"
        "with tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), 2048) as rt:\n"
        "    for _ in range(2):\n"
        "        rt.multiply(A, B, a_uid='A', b_uid='B', out=C)\n"
        "np.save(sys.argv[1], C.cpu().numpy())\n"
        "print('dies', tr.dense.k1_die_map(0))\n")
    root = Path(__file__).resolve().parents[1]
    outs = {}
    for flag in ("1", "0"):
        f = tmp_path / f"c{flag}.npy"
        env = dict(os.environ, TR_K1_DIE=flag, PYTHONPATH=str(root))
        r = subprocess.run([sys.executable, "-c", code, str(f)], capture_output=True, text=True, env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[flag] = (np.load(f), r.stdout)
    assert "dies (0, 0)" in outs["0"][1] and "dies (0, 0)" not in outs["1"][1]
    assert np.array_equal(outs["1"][0], outs["0"][0])


@pytest.mark.parametrize("shape", [(0, 5, 4), (4, 5, 0), (4, 0, 3)])
def test_empty_dimensions_are_a_value_error(shape):
    """As the reference's matrices (tiles.py as_matrix): a zero dimension is a
    ValueError, on the dense path and through run()."""
    import numpy as np

    from paper_1511_04348_b200 import homogeneous_machine, run

    m, k, n = shape
    a, b = np.zeros((m, k)), np.zeros((k, n))
    with pytest.raises(ValueError):
        run(homogeneous_machine(1), a, b, 4)
    with pytest.raises(ValueError):
        dense_gemm(torch.zeros((m, k), device="cuda"), torch.zeros((k, n), device="cuda"))


@pytest.mark.parametrize("precision", ["fp32acc", "fp32hi", "bf16", "exact"])
def test_inf_and_nan_propagate_like_numpy(precision):
    """Non-finite inputs give non-finite outputs exactly where the reference's
    are, and NaN where it has NaN, in every mode.  An inf stays inf in the bf16
    and exact modes; the split modes (fp32acc, fp32hi) keep inf in the hi plane
    (lo = 0, not inf - inf) but the cross product inf x lo of the other operand
    is -inf wherever that lo is negative, so about half of such outputs become
    NaN.  Every finite element stays within tolerance."""
    import numpy as np

    from paper_1511_04348_b200 import homogeneous_machine, run

    rng = np.random.default_rng(2)
    a = rng.standard_normal((300, 200)).astype(np.float32)
    b = np.abs(rng.standard_normal((200, 260))).astype(np.float32) + 0.1
    a[5, 7] = np.inf
    a[9, 3] = np.nan
    ref = a.astype(np.float64) @ b.astype(np.float64)
    for c in (run(homogeneous_machine(1, dtype=np.float32), a, b, 128, precision=precision)[0],
              dense_gemm(torch.as_tensor(a).cuda(), torch.as_tensor(b).cuda(), precision=precision).cpu().numpy()):
        assert np.array_equal(np.isfinite(c), np.isfinite(ref)) and np.isnan(c[np.isnan(ref)]).all()
        if precision in ("bf16", "exact"):
            assert np.array_equal(np.isinf(c), np.isinf(ref))
            assert np.array_equal(np.sign(c[np.isinf(ref)]), np.sign(ref[np.isinf(ref)]))
        else:
            assert np.isinf(c[np.isinf(ref)]).any()
        fin = np.isfinite(ref)
        tol = {"fp32acc": 1e-5, "fp32hi": 2e-6, "bf16": 1e-2, "exact": 1e-6}[precision]
        assert np.linalg.norm(c[fin] - ref[fin]) <= tol * np.linalg.norm(ref[fin])
