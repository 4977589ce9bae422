"""The CUDA-core task GEMM (csrc/small_gemm.cu): narrow output tiles (n <= 32,
e.g. the MLP's 10-wide output layer) and tiny contractions (k <= 32, its
dX = dY W^T) through the runtime, against float64 references, against the
tensor-core kernel, and bit-exact on integer inputs."""

import numpy as np
import pytest
import torch
from torch.profiler import ProfilerActivity, profile

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import Runtime, homogeneous_machine, run
from paper_1511_04348_b200.dense import set_narrow_tc, set_small_gemm, set_splitk

pytestmark = pytest.mark.gpu


def rel(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / np.linalg.norm(ref))


@pytest.fixture
def small():
    yield set_small_gemm
    set_small_gemm(True)
    set_narrow_tc(True)
    set_splitk(8)


def kernels_run(fn):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events() if e.device_type.name == "CUDA"}


SHAPES = [  # m, k, n, tile, transpose_a, transpose_b
    (4096 + 300, 9000, 10, 4096, False, False),  # the output layer's forward product, ragged rows
    (1000, 3000, 32, 512, True, False),          # its dW = X^T dY (transposed A)
    (777, 5000, 17, 1024, False, True),
    (3000, 10, 2000, 1024, False, True),         # dX = dY W^T: tiny contraction, transposed B
    (500, 32, 700, 256, True, True),
    (300, 7, 5000, 4096, False, False),
]


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
@pytest.mark.parametrize("m,k,n,tile,ta,tb", SHAPES)
def test_matches_f64_and_tensor_cores(small, precision, m, k, n, tile, ta, tb):
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
    ref = (a.double().T if ta else a.double()) @ (b.double().T if tb else b.double())
    outs = {}
    narrow = n <= 32 and k > 32
    # default: narrow tiles as the transposed tensor-core product, tiny contractions
    # on CUDA cores; "cuda": narrow tiles on CUDA cores too; "tc": everything on
    # the tensor cores in the plain orientation
    for mode in ("default", "cuda", "tc"):
        small(mode != "tc")
        set_narrow_tc(mode == "default")
        rt = Runtime(homogeneous_machine(1, dtype=np.float32), tile, precision=precision)
        c = torch.empty(m, n, device="cuda")
        names = kernels_run(lambda: rt.multiply(a, b, transpose_a=ta, transpose_b=tb, out=c))
        used_small = any("small_gemm" in x for x in names)
        used_t = any("reduce_t" in x for x in names)
        if mode == "default":
            assert used_t == narrow and used_small == (not narrow), names
        elif mode == "cuda":
            assert used_small and not used_t, names
        else:
            assert not used_small and not used_t, names
        outs[mode] = c.double()
        rt.close()
    tol = 1e-5 if precision == "fp32acc" else 1e-2
    for c in outs.values():
        assert rel(c.cpu().numpy(), ref.cpu().numpy()) <= tol
    assert rel(outs["default"].cpu().numpy(), outs["tc"].cpu().numpy()) <= tol


@pytest.mark.parametrize("m,k,n,tile,cap", [(700, 4000, 10, 256, None), (600, 12, 900, 256, None),
                                             (300, 2000, 30, 128, 5)])
def test_integer_exact_split_and_chunked(small, m, k, n, tile, cap):
    """Integer inputs make every order exact: the CUDA-core result (split-K,
    and chunked k-steps accumulating into C when cap=5) equals the oracle."""
    rng = np.random.default_rng(m * n)
    a = rng.integers(-4, 5, size=(m, k)).astype(np.float64)
    b = rng.integers(-4, 5, size=(k, n)).astype(np.float64)
    machine = homogeneous_machine(2, capacity_tiles=cap)
    for splits, narrow in ((8, True), (1, True), (8, False)):
        set_splitk(splits)
        set_narrow_tc(narrow)
        c, s = run(machine, a, b, tile)
        assert np.array_equal(c, O.reference_gemm(a, b))
        assert s.cache.input_requests == 2 * s.total_tasks * -(-k // tile)


def test_fused_posts_and_write_through():
    """The output layer's round trip: forward (bias + sigmoid, 10 wide), dX with
    act_grad written through into the tile cache, then a product reading that
    cached result -- equal to the same chain with write-through off."""
    g = torch.Generator().manual_seed(4)
    f = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)
    x, w, bias, dy = f(2048, 1024), f(1024, 10), f(10), f(2048, 10)
    a_prev = torch.rand(2048, 1024, generator=g, dtype=torch.float64)
    dev = lambda t: t.float().cuda().contiguous()
    res = []
    for wt in ("DY", None):
        rt = Runtime(homogeneous_machine(1, dtype=np.float32), 1024)
        fwd = torch.empty(2048, 10, device="cuda")
        dx = torch.empty(2048, 1024, device="cuda")
        rt.multiply_batch([dict(a=dev(x), b=dev(w), out=fwd, post=("bias_act", dev(bias), "sigmoid"))])
        rt.multiply_batch([dict(a=dev(dy), b=dev(w), out=dx, transpose_b=True, post=("act_grad", dev(a_prev), "sigmoid"),
                                cache_as=wt)])
        dw = torch.empty(1024, 1024, device="cuda")
        rt.multiply(dev(x), dx, transpose_a=True, out=dw, a_uid="X", b_uid=wt)
        res.append((fwd.double().cpu(), dx.double().cpu(), dw.double().cpu()))
        rt.close()
    r32 = lambda t: t.float().double()
    ref_f = torch.sigmoid(r32(x) @ r32(w) + r32(bias))
    ref_dx = (r32(dy) @ r32(w).T) * (r32(a_prev) * (1 - r32(a_prev)))
    assert rel(res[0][0].numpy(), ref_f.numpy()) <= 5e-5
    assert rel(res[0][1].numpy(), ref_dx.numpy()) <= 1e-5
    for u, v in zip(res[0], res[1]):
        assert torch.equal(u, v)


@pytest.mark.parametrize("m,k,n,tile,ta", [(700, 4000, 10, 256, True), (1000, 3000, 700, 256, True),
                                            (2048, 2048, 2048, 1024, True), (600, 12, 900, 256, False)])
def test_axpy_products(m, k, n, tile, ta):
    """out += alpha * a.b (the fused SGD update W += (-lr) X^T dY) on every
    kernel path: CUDA-core (narrow, split), tensor-core (single / grouped,
    split-K) -- against float64."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
    b = torch.randn(k, n, device="cuda", generator=g)
    w = torch.randn(m, n, device="cuda", generator=g)
    ref = w.double() - 0.125 * ((a.double().T if ta else a.double()) @ b.double())
    rt = Runtime(homogeneous_machine(1, dtype=np.float32), tile)
    rt.multiply_batch([dict(a=a, b=b, out=w, transpose_a=ta, axpy=-0.125)])
    assert rel(w.double().cpu().numpy(), ref.cpu().numpy()) <= 1e-5
    rt.close()
