"""The scheduled GPU product (tr_gemm through Runtime/run) against the oracle
and the reference's golden runs.

Tolerances (north star): integer-valued inputs are exact (they are exactly
representable in bf16 and the sums in fp32); float inputs <= 1e-5 relative
Frobenius error in the fp32-accurate mode, <= 1e-2 in bf16 mode.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix, Runtime, homogeneous_machine, run

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
TOL = {"fp32acc": 1e-5, "bf16": 1e-2}


def rel(c, ref):
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(np.asarray(c, np.float64) - ref) / (den if den else 1.0))


def int_matrix(rng, r, c):
    return rng.integers(-4, 5, size=(r, c)).astype(np.float64)


@pytest.fixture(scope="module")
def golden():
    return json.loads((G / "runs.json").read_text()), np.load(G / "runs.npz")


def test_golden_runs(golden):
    meta, arr = golden
    for name, m in meta.items():
        if name in ("session_reuse", "transpose"):
            continue
        a, b, cref = arr[name + "_a"], arr[name + "_b"], arr[name + "_c"]
        c, s = run(homogeneous_machine(m["devices"], capacity_tiles=m["capacity"]), a, b, m["tile"],
                   coherence=m["coherence"], directory_debug=True)
        if m["kind"] == "int":
            assert np.array_equal(c, cref), (name, np.argwhere(c != cref)[:5].tolist())
        else:
            d = np.abs(c - cref)
            worst = np.unravel_index(np.argmax(d), d.shape)
            assert rel(c, cref) <= TOL["fp32acc"], (name, rel(c, cref), worst, c[worst], cref[worst],
                                                    int((d > 1e-3 * np.abs(cref).max()).sum()))
        assert c.dtype == cref.dtype
        ref_cache = m["stats"]["cache"]
        assert s.total_tasks == m["stats"]["total_tasks"] == sum(s.tasks_by_device.values())
        assert s.cache.input_requests == ref_cache["l1_hits"] + ref_cache["l2_hits"] + ref_cache["host_fetches"]
        assert s.cache.writebacks == ref_cache["writebacks"]
        if m["devices"] == 1:
            assert s.cache.as_dict() == ref_cache, name  # deterministic one-device schedule
        elif m["capacity"] is None:
            assert s.cache.host_fetches == ref_cache["host_fetches"], name
        assert s.gpu_launches > 0


def test_session_reuse_and_transpose(golden):
    meta, arr = golden
    a, b = arr["session_reuse_a"], arr["session_reuse_b"]
    rt = Runtime(homogeneous_machine(1), 4)
    c1, s1 = rt.multiply(a, b, a_uid="X", b_uid="W")
    c2, s2 = rt.multiply(a, b, a_uid="X", b_uid="W")
    assert s1.cache.as_dict() == meta["session_reuse"]["first"]["cache"]
    assert s2.cache.as_dict() == meta["session_reuse"]["second"]["cache"]
    assert np.array_equal(c1, O.reference_gemm(a, b)) and np.array_equal(c1, c2)
    x, w, y = arr["transpose_x"], arr["transpose_w"], arr["transpose_y"]
    rt = Runtime(homogeneous_machine(1), 4)
    rt.multiply(x, w, a_uid="X", b_uid="W")
    before = rt.directory.stats()
    c, _ = rt.multiply(x, y, transpose_a=True, a_uid="X", b_uid="Y2")
    assert rt.directory.stats().host_fetches - before.host_fetches == meta["transpose"]["host_fetch_delta"]
    assert rel(c, arr["transpose_c"]) <= 1e-5


def test_c1_randomized_cases():
    """Acceptance C1 (reference test_acceptance.py:56-92), checked against the oracle."""
    rng = np.random.default_rng(20240601)
    dim_hi = {1: 24, 7: 256, 16: 512, 64: 512}
    for case in range(30):
        t = int(rng.choice([1, 7, 16, 64]))
        m, k, n = (int(rng.integers(1, dim_hi[t] + 1)) for _ in range(3))
        ndev = int(rng.choice([1, 2, 4]))
        kind = "int" if case % 2 else "float"
        if kind == "int":
            a, b = int_matrix(rng, m, k), int_matrix(rng, k, n)
        else:
            a, b = rng.uniform(0.0, 1.0, size=(m, k)), rng.uniform(0.0, 1.0, size=(k, n))
        c, s = run(homogeneous_machine(ndev), a, b, t)
        ref = O.c_oracle().gemm(a, b)
        label = f"{m}x{k}x{n} T={t} dev={ndev} {kind}"
        if kind == "int":
            assert np.array_equal(c, ref), label
        else:
            assert rel(c, ref) <= 1e-5, label
        assert sum(s.tasks_by_device.values()) == s.total_tasks


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_transposed_operands_normal_data(precision, ta, tb):
    rng = np.random.default_rng(3)
    m, k, n, t = 300, 520, 270, 128
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    rt = Runtime(homogeneous_machine(2), t, precision=precision)
    c, s = rt.multiply(a, b, transpose_a=ta, transpose_b=tb)
    ref = O.reference_gemm(a.T if ta else a, b.T if tb else b)
    assert rel(c, ref) <= TOL[precision]


def test_float32_machine_and_device_resident_operands():
    rng = np.random.default_rng(4)
    a = rng.standard_normal((700, 900)).astype(np.float32)
    b = rng.standard_normal((900, 500)).astype(np.float32)
    m = homogeneous_machine(2, dtype=np.float32)
    c_host, s = run(m, a, b, 256)
    assert c_host.dtype == np.float32
    assert s.cache.bytes_host == (700 * 900 + 900 * 500) * 4  # each distinct tile crosses PCIe once
    ref = O.c_oracle().gemm(a.astype(np.float64), b.astype(np.float64))
    assert rel(c_host, ref) <= 1e-5
    rt = Runtime(m, 256)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c_dev, _ = rt.multiply(ta, tb)
    assert c_dev.is_cuda and c_dev.dtype == torch.float32
    assert np.array_equal(c_dev.cpu().numpy(), c_host)  # same tiles, same kernel, same order


def test_capacity_three_exact_with_evictions():
    rng = np.random.default_rng(8)
    a, b = int_matrix(rng, 40, 40), int_matrix(rng, 40, 40)
    c, s = run(homogeneous_machine(2, capacity_tiles=3), a, b, 5, directory_debug=True)
    assert np.array_equal(c, O.reference_gemm(a, b))
    assert s.cache.evictions > 0 and s.cache.input_requests == 2 * s.total_tasks * s.k_steps


def test_exactly_once_threaded_stress():
    rng = np.random.default_rng(7)
    for _ in range(20):
        t, g = int(rng.integers(3, 6)), int(rng.integers(2, 5))
        ndev = int(rng.integers(2, 5))
        a, b = int_matrix(rng, t * g, t * g), int_matrix(rng, t * g, t * g)
        c, s = run(homogeneous_machine(ndev), a, b, t, directory_debug=True)
        assert np.array_equal(c, O.reference_gemm(a, b))
        assert sum(s.tasks_by_device.values()) == s.total_tasks == g * g


def test_peer_hits_and_heterogeneous_slots():
    rng = np.random.default_rng(9)
    a, b = int_matrix(rng, 96, 96), int_matrix(rng, 96, 96)
    devs = [DeviceSpec(0, slots=1), DeviceSpec(1, slots=4), DeviceSpec(2, slots=2)]
    m = Machine(devs, ProximityMatrix.uniform(3))
    c, s = run(m, a, b, 16)
    assert np.array_equal(c, O.reference_gemm(a, b))
    assert s.cache.host_fetches == 2 * 6 * 6 and s.cache.l2_hits > 0
    assert s.cache.bytes_peer == s.cache.l2_hits * 16 * 16 * 8


def test_bypass_mode_counts_and_result():
    rng = np.random.default_rng(10)
    a, b = int_matrix(rng, 24, 24), int_matrix(rng, 24, 24)
    c, s = run(homogeneous_machine(2), a, b, 4, coherence=False)
    assert np.array_equal(c, O.reference_gemm(a, b)) and s.cache.host_fetches == 2 * 6 ** 3


def test_reports_kernel_time():
    rng = np.random.default_rng(11)
    a, b = rng.standard_normal((1024, 1024)), rng.standard_normal((1024, 1024))
    _, s = run(homogeneous_machine(1), a, b, 512)
    assert s.kernel_ms[0] > 0 and s.wall_elapsed > 0


def test_first_touch_identity_with_fetch_ahead_under_stealing():
    """Fetch-ahead must not change any counter: across many multi-device runs
    (where stealing moves reserved tasks whose tiles were already fetched
    ahead), every distinct tile is still counted as exactly one host fetch."""
    rng = np.random.default_rng(21)
    for trial in range(25):
        t, g, ndev = 8, int(rng.integers(3, 7)), int(rng.integers(2, 5))
        a, b = int_matrix(rng, t * g, t * g), int_matrix(rng, t * g, t * g)
        c, s = run(homogeneous_machine(ndev, dtype=np.float64), a, b, t, directory_debug=True)
        assert np.array_equal(c, O.reference_gemm(a, b))
        assert s.cache.host_fetches == 2 * g * g, (trial, ndev, s.cache)
        assert s.cache.bytes_host == 2 * g * g * t * t * 8
        assert s.cache.input_requests == 2 * g ** 3
        assert s.cache.bytes_peer == s.cache.l2_hits * t * t * 8


@pytest.mark.parametrize("act", ["sigmoid", "relu", "identity"])
def test_batch_with_fused_epilogues(act):
    """tr_gemm_batch: independent products in one round, with the fused MLP
    post-ops (bias + activation; times act'(a)) against a float64 torch reference."""
    g = torch.Generator().manual_seed(5)
    f = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)
    x, w, bias, dy = f(300, 520), f(520, 270), f(270), f(300, 270)
    a_prev = torch.rand(300, 520, generator=g, dtype=torch.float64)  # an activation output
    if act == "relu":
        a_prev = torch.relu(a_prev - 0.5)
    dev = lambda t: t.float().cuda().contiguous()
    out1 = torch.empty(300, 270, device="cuda")
    out2 = torch.empty(300, 520, device="cuda")
    rt = Runtime(homogeneous_machine(2, dtype=np.float32), 128)
    s = rt.multiply_batch([
        dict(a=dev(x), b=dev(w), out=out1, post=("bias_act", dev(bias), act)),
        dict(a=dev(dy), b=dev(w), out=out2, transpose_b=True, post=("act_grad", dev(a_prev), act)),
    ])
    fwd = {"sigmoid": torch.sigmoid, "relu": torch.relu, "identity": lambda v: v}[act]
    grad = {"sigmoid": lambda a: a * (1 - a), "relu": lambda a: (a > 0).double(),
            "identity": lambda a: torch.ones_like(a)}[act]
    ref1 = fwd(x @ w + bias)
    ref2 = (dy @ w.T) * grad(a_prev.float().double())
    assert rel(out1.double().cpu().numpy(), ref1.numpy()) <= 1e-5
    assert rel(out2.double().cpu().numpy(), ref2.numpy()) <= 1e-5
    assert s.total_tasks == 3 * 3 + 3 * 5
    rt.close()


@pytest.mark.parametrize("tile", [128, 16])
def test_fused_epilogue_operands_with_odd_strides(tile):
    """Fused post-op operands need not be 16-byte aligned: an activation that is
    a column slice of a wider buffer (row stride 523 floats, offset 1) feeds the
    act_grad epilogue of both kernels (tile 128: tensor cores; 16: CUDA cores)."""
    g = torch.Generator().manual_seed(13)
    dy, w = torch.randn(300, 270, generator=g, dtype=torch.float64), torch.randn(520, 270, generator=g, dtype=torch.float64)
    wide = torch.rand(300, 523, generator=g, dtype=torch.float64)
    a_prev = wide[:, 1:521]
    dev = lambda t: t.float().cuda().contiguous()
    aux = wide.float().cuda()[:, 1:521]
    assert aux.stride(0) == 523 and aux.data_ptr() % 16 != 0
    out = torch.empty(300, 520, device="cuda")
    rt = Runtime(homogeneous_machine(1, dtype=np.float32), tile)
    rt.multiply_batch([dict(a=dev(dy), b=dev(w), out=out, transpose_b=True, post=("act_grad", aux, "sigmoid"))])
    r32 = lambda t: t.float().double()
    ref = (r32(dy) @ r32(w).T) * (r32(a_prev) * (1 - r32(a_prev)))
    assert rel(out.double().cpu().numpy(), ref.numpy()) <= 1e-5
    rt.close()


@pytest.mark.parametrize("side", [True, False])
def test_stream_ordered_chain_with_torch_ops(side):
    """Runtime.set_stream(ordered=True): products return once enqueued; a chain
    product -> torch op -> product on the same stream (a side stream, or the
    legacy default stream) sees every prior result, and matches the blocking run
    bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(700, 500, device="cuda", generator=g)
    b = torch.randn(500, 500, device="cuda", generator=g)
    outs = {}
    for ordered in (False, True):
        rt = Runtime(homogeneous_machine(2, dtype=np.float32, gpus=[0, 0]), 128)
        stream = torch.cuda.Stream() if side else torch.cuda.default_stream()
        stream.wait_stream(torch.cuda.current_stream())  # a, b were made on the default stream
        rt.set_stream(stream, ordered=ordered)
        with torch.cuda.stream(stream):
            c = a.clone()
            for step in range(5):
                nxt = torch.empty_like(c)
                s = rt.multiply(c, b, out=nxt, a_uid=f"c{step}", b_uid="B")[1]
                assert s.total_tasks == 6 * 4 and s.cache.writebacks == 24
                c = torch.tanh(nxt * 0.05)  # torch kernel on the same stream, reads the product
        stream.synchronize()
        outs[ordered] = c.cpu()
        ref = a.double()
        for _ in range(5):
            ref = torch.tanh((ref @ b.double()) * 0.05)
        assert rel(c.double().cpu().numpy(), ref.cpu().numpy()) <= 5 * 1e-5  # five chained products
        rt.close()
    assert torch.equal(outs[True], outs[False])


@pytest.fixture
def no_split():
    from paper_1511_04348_b200.dense import set_splitk

    yield lambda on: set_splitk(1 if on else 8)
    set_splitk(8)


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
@pytest.mark.parametrize("m,k,n,tile,cap", [(300, 5000, 10, 512, None), (200, 3000, 700, 1024, None),
                                             (130, 2600, 40, 256, 5)])
def test_split_k_exact_on_integers(no_split, precision, m, k, n, tile, cap):
    """Skinny outputs run split-K (partials reduced in a fixed order); integer
    inputs make every summation order exact, so split and unsplit agree bitwise
    (cap=5 also forces chunked launches that accumulate into C)."""
    rng = np.random.default_rng(m + n)
    a, b = int_matrix(rng, m, k), int_matrix(rng, k, n)
    machine = homogeneous_machine(2, capacity_tiles=cap)
    outs = []
    for off in (False, True):
        no_split(off)
        c, s = run(machine, a, b, tile, precision=precision)
        outs.append(c)
    assert np.array_equal(outs[0], O.reference_gemm(a, b))
    assert np.array_equal(outs[0], outs[1])


@pytest.fixture
def tensor_cores_only():
    """Every task on the tensor-core kernel in its plain orientation (no CUDA-core
    or transposed narrow path): the split-K tests below are about that kernel."""
    from paper_1511_04348_b200.dense import set_narrow_tc, set_small_gemm

    set_small_gemm(False)
    set_narrow_tc(False)
    yield
    set_small_gemm(True)
    set_narrow_tc(True)


def test_split_k_normal_data_and_fused_posts(no_split, tensor_cores_only):
    g = torch.Generator().manual_seed(11)
    f = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)
    x, w, bias = f(1000, 8192), f(8192, 10), f(10)
    dy, w2 = f(1000, 10), f(784, 10)
    a_prev = torch.rand(1000, 784, generator=g, dtype=torch.float64)
    dev = lambda t: t.float().cuda().contiguous()
    res = {}
    for off in (False, True):
        no_split(off)
        rt = Runtime(homogeneous_machine(1, dtype=np.float32), 4096)
        o1 = torch.empty(1000, 10, device="cuda")
        o2 = torch.empty(1000, 784, device="cuda")
        s = rt.multiply_batch([dict(a=dev(x), b=dev(w), out=o1, post=("bias_act", dev(bias), "sigmoid")),
                               dict(a=dev(dy), b=dev(w2), out=o2, transpose_b=True,
                                    post=("act_grad", dev(a_prev), "sigmoid"))])
        assert s.total_tasks == 2
        res[off] = (o1.double().cpu(), o2.double().cpu(), s.gpu_launches)
        rt.close()
    r32 = lambda t: t.float().double()  # the operands the GPU actually sees
    ref1 = torch.sigmoid(r32(x) @ r32(w) + r32(bias))
    ref2 = (r32(dy) @ r32(w2).T) * (r32(a_prev) * (1 - r32(a_prev)))
    # pre-activations here are ~N(0, 8192): the product's 1e-5 relative error is
    # relative to that scale, and the sigmoid (which maps it into (0, 1)) amplifies
    # it in relative terms, hence 5e-5 for the fused output
    for o1, o2, _ in res.values():
        assert rel(o1.numpy(), ref1.numpy()) <= 5e-5
        assert rel(o2.numpy(), ref2.numpy()) <= 1e-5
    assert rel(res[False][0].numpy(), res[True][0].numpy()) <= 1e-5  # split vs unsplit: summation order only
    assert res[False][2] > res[True][2]  # the split run launched reduction kernels


@pytest.fixture
def task_group():
    from paper_1511_04348_b200.dense import set_task_group

    yield set_task_group
    set_task_group(4)


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_grouped_launches_match_single(task_group, precision, ta, tb):
    """Device-resident products run up to 4 station tasks per K1 launch; every
    tile is computed by the same code, so grouped and per-task launches agree
    bit for bit, with the reference's counters and one writeback per task."""
    g = torch.Generator(device="cuda").manual_seed(21)
    m, k, n = 1000, 700, 1100
    a = torch.randn(k if ta else m, m if ta else k, device="cuda", generator=g)
    b = torch.randn(n if tb else k, k if tb else n, device="cuda", generator=g)
    outs = {}
    for grp in (1, 4):
        task_group(grp)
        rt = Runtime(homogeneous_machine(2, dtype=np.float32, gpus=[0, 0]), 256, precision=precision)
        c = torch.empty(m, n, device="cuda")
        _, s = rt.multiply(a, b, transpose_a=ta, transpose_b=tb, a_uid="A", b_uid="B", out=c)
        gm, gn, gk = -(-m // 256), -(-n // 256), -(-k // 256)
        assert s.total_tasks == gm * gn and s.cache.writebacks == gm * gn
        assert s.cache.l1_hits + s.cache.l2_hits + s.cache.host_fetches == 2 * gm * gn * gk
        outs[grp] = (c.cpu(), s.gpu_launches)
        rt.close()
    assert torch.equal(outs[1][0], outs[4][0])
    assert outs[4][1] < outs[1][1]  # fewer launches when grouped
    ref = (a.double().T if ta else a.double()) @ (b.double().T if tb else b.double())
    assert rel(outs[4][0].double().numpy(), ref.cpu().numpy()) <= TOL[precision]


def test_grouped_launches_with_fused_posts_and_mlp(task_group):
    """The MLP's fused epilogues in grouped launches: bitwise equal to per-task."""
    rng = np.random.default_rng(4)
    sizes = [300, 1100, 900, 7]
    from paper_1511_04348_b200 import GpuMLP, Layer

    base = [Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}") for i in range(3)]
    x, t = O.random_regression(rng, 600, 300, 7)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    res = {}
    for grp in (1, 4):
        task_group(grp)
        layers = [Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base]
        mlp = GpuMLP(layers, tile_size=256)
        res[grp] = ([mlp.train_step(xd, td, 0.3) for _ in range(3)], mlp.to_host())
        mlp.close()
    assert res[1][0] == res[4][0]
    for (w1, b1), (w4, b4) in zip(res[1][1], res[4][1]):
        assert np.array_equal(w1, w4) and np.array_equal(b1, b4)


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
def test_kpanel_schedule_cold_product(precision):
    """A cold single-device product (host A, B, C) runs the k-panel schedule:
    the reference's counters exactly, integer inputs exact, float inputs within
    tolerance, and the same numbers as the shells order up to rounding."""
    rng = np.random.default_rng(31)
    m, k, n, T = 1100, 1500, 900, 128  # 9 x 8 tasks, 12 k-steps
    ai, bi = int_matrix(rng, m, k), int_matrix(rng, k, n)
    af, bf = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    gm, gn, gk = -(-m // T), -(-n // T), -(-k // T)
    res = {}
    for order in ("auto", "shells"):
        rt = Runtime(homogeneous_machine(1), T, precision=precision)
        rt.set_order(order)
        ci, s = rt.multiply(ai, bi, a_uid="Ai", b_uid="Bi")
        assert np.array_equal(ci, O.reference_gemm(ai, bi))
        assert s.cache.host_fetches == gm * gk + gk * gn and s.cache.writebacks == gm * gn
        assert s.cache.l1_hits == 2 * gm * gn * gk - (gm * gk + gk * gn)
        assert s.tasks_by_device == {0: gm * gn}
        cf, _ = rt.multiply(af, bf, a_uid="Af", b_uid="Bf")
        assert rel(cf, af @ bf) <= TOL[precision]
        res[order] = cf
        rt.close()
    assert rel(res["auto"], res["shells"]) <= 1e-6 if precision == "fp32acc" else 1e-3


def test_host_output_grouped_launches():
    """Tasks with HOST outputs run as grouped launches (C tiles in the stream's
    group buffer, written back on the writeback stream): non-persistent while
    host tiles are still being filled (cold), persistent once every input is
    resident (warm re-multiply).  Integer inputs are exact, ragged edges
    included; both runs give the same bits and the reference's counters."""
    rng = np.random.default_rng(41)
    m, k, n, T = 1100, 1300, 1000, 256  # 5 x 4 tasks, 6 k-steps, ragged edges
    a, b = int_matrix(rng, m, k).astype(np.float32), int_matrix(rng, k, n).astype(np.float32)
    gm, gn, gk = -(-m // T), -(-n // T), -(-k // T)
    ref = O.reference_gemm(a.astype(np.float64), b.astype(np.float64))
    def gemm_launches(stats):  # tasks of one grouped launch share its timing events
        ev = [e for e in stats.trace if e["kind"] == "gemm"]
        assert len(ev) == gm * gn
        return len({(e["start_ms"], e["end_ms"]) for e in ev})

    with Runtime(homogeneous_machine(1, dtype=np.float32), T, trace=True) as rt:
        rt.set_order("shells")  # the task path (not the k-panel schedule)
        c1, s1 = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C1")
        assert np.array_equal(c1, ref)
        assert s1.cache.host_fetches == gm * gk + gk * gn and s1.cache.writebacks == gm * gn
        assert gemm_launches(s1) < gm * gn
        c2, s2 = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C2")
        assert s2.cache.host_fetches == 0 and s2.cache.writebacks == gm * gn
        assert gemm_launches(s2) < gm * gn
        assert np.array_equal(c1, c2)
        assert s2.tasks_by_device == {0: gm * gn}


def test_host_slices_read_in_place():
    """Row slices of A, column slices of B and a sub-block of C are read and
    written in place (pitched copies with the parent's row stride)."""
    rng = np.random.default_rng(12)
    a, b = int_matrix(rng, 700, 520), int_matrix(rng, 520, 900)
    c = np.full((700, 900), -7.0)
    a_v, b_v, c_v = a[100:600], b[:, 250:830], c[100:600, 250:830]
    assert not b_v.flags.c_contiguous
    rt = Runtime(homogeneous_machine(2, gpus=[0, 0]), 128)
    out, s = rt.multiply(a_v, b_v, out=c_v)
    assert out is c_v
    assert np.array_equal(c[100:600, 250:830], O.reference_gemm(a_v, b_v))
    assert (c[:100] == -7).all() and (c[:, :250] == -7).all() and (c[600:] == -7).all() and (c[:, 830:] == -7).all()
    rt.close()


def test_green_context_devices_balance_load():
    """Two logical devices on one B200 with disjoint green-context SM groups
    (64 and 32 SMs): the product is exact on integer inputs and the dynamic
    scheduler (queue + stations + stealing) hands the faster device about twice
    the tasks -- the reference's inhomogeneous-devices acceptance behaviour
    (tests/test_acceptance.py:130-141) on real hardware."""
    from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix

    rng = np.random.default_rng(50)
    n, T = 16384, 2048  # 64 tasks, each long enough (~0.8 / 1.6 ms) for the split to show
    a = rng.integers(-4, 5, size=(n, n)).astype(np.float32)
    b = rng.integers(-4, 5, size=(n, n)).astype(np.float32)
    m = Machine([DeviceSpec(0, gpu=0, sms=64), DeviceSpec(1, gpu=0, sms=32)], ProximityMatrix.uniform(2),
                dtype=np.float32)
    rt = Runtime(m, T)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c = torch.empty(n, n, device="cuda")
    rt.multiply(ad, bd, a_uid="A", b_uid="B", out=c)  # warm: tiles resident on whichever device took them
    counts = []
    for _ in range(3):
        _, s = rt.multiply(ad, bd, a_uid="A", b_uid="B", out=c)
        counts.append((s.tasks_by_device[0], s.tasks_by_device[1]))
    ref = O.c_oracle().gemm(a[:8].astype(np.float64), b.astype(np.float64))
    assert np.array_equal(c[:8].double().cpu().numpy(), ref)
    fast, slow = map(sum, zip(*counts))
    assert fast + slow == 3 * 64
    assert 1.4 <= fast / slow <= 2.8, counts  # 64 : 32 SMs
    rt.close()


def test_green_context_devices_1234():
    """Four green-context devices of 8 / 16 / 24 / 32 SMs on one GPU share a
    product of a 32 x 32 task grid (the reference's acceptance shape,
    test_acceptance.py:130-141): each device's share of the work is within 10 %
    (relative) of its share of the devices' measured standalone throughputs."""
    from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix, standalone_rates

    n, T = 32768, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(n, n, device="cuda", generator=g)
    b = torch.randn(n, n, device="cuda", generator=g)
    c = torch.empty(n, n, device="cuda")
    m = Machine([DeviceSpec(i, gpu=0, sms=8 * (i + 1)) for i in range(4)], ProximityMatrix.uniform(4),
                dtype=np.float32)
    rates = np.array(standalone_rates(m, T, a[: 8 * T], b, out=c[: 8 * T]))
    assert np.all(np.diff(rates) > 0)  # more SMs, more throughput
    rt = Runtime(m, T)
    rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
    _, s = rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
    assert s.total_tasks == 1024 == sum(s.tasks_by_device.values())
    work = np.array([s.devices[d].macs for d in range(4)], dtype=np.float64)
    assert work.sum() == float(n) ** 3
    share, ideal = work / work.sum(), rates / rates.sum()
    assert np.all(np.abs(share - ideal) <= 0.10 * ideal), (share, ideal)
    rows = torch.arange(0, n, 997, device="cuda")
    ref = a[rows].double() @ b.double()
    assert rel(c[rows].double().cpu().numpy(), ref.cpu().numpy()) <= 1e-5
    rt.close()


def test_standalone_rates_follow_sm_counts():
    """standalone_rates: each device's throughput alone; identical specs are
    measured once, and an 8-SM green context runs at about half a 16-SM one."""
    from paper_1511_04348_b200 import standalone_rates

    T = 1024
    a = torch.randn(8 * T, 8 * T, device="cuda")
    b = torch.randn(8 * T, 8 * T, device="cuda")
    c = torch.empty(8 * T, 8 * T, device="cuda")
    m = Machine([DeviceSpec(0, gpu=0, sms=16), DeviceSpec(1, gpu=0, sms=8), DeviceSpec(2, gpu=0, sms=16)],
                ProximityMatrix.uniform(3), dtype=np.float32)
    # a 1.1 TFLOP product (tens of ms per device): the rates of small green
    # contexts follow the boost clock, which a preceding heavy test can lower
    r = standalone_rates(m, T, a, b, out=c, reps=3)
    assert r[0] == r[2] and 0.3 <= r[1] / r[0] <= 0.75, r


def test_execute_task_by_hand_state_machine():
    """scheduler._execute_task (the reference's internal helper, scheduler.py:371-410)
    driven by hand with plan / ReservationStation / CacheDirectory: every task
    QUEUED -> RESERVED -> DONE, the product exact, a second mark refused."""
    from paper_1511_04348_b200 import CacheDirectory, ReservationStation, TaskState, partition, plan, reassemble
    from paper_1511_04348_b200.scheduler import _execute_task

    rng = np.random.default_rng(16)
    a, b = int_matrix(rng, 12, 8), int_matrix(rng, 8, 12)
    machine = homogeneous_machine(1)
    p = plan(partition(a, 4), partition(b, 4))
    directory = CacheDirectory(machine, debug=True)
    st = ReservationStation(0, 4)
    steps_total = 0
    while not p.queue.is_empty():
        for tid in st.refill(p.queue):
            p.tasks[tid].state = TaskState.RESERVED
        while (tid := st.pop_for_run()) is not None:
            steps, wb = _execute_task(machine, p, directory, machine.device(0), p.tasks[tid])
            steps_total += len(steps)
            assert wb > 0
    assert all(t.state is TaskState.DONE for t in p.tasks) and steps_total == 9 * 2
    assert np.array_equal(reassemble(p.c.tiled), O.reference_gemm(a, b))
    assert directory.stats().host_fetches == 3 * 2 + 2 * 3
    with pytest.raises(RuntimeError):
        p.completion.mark(0)
