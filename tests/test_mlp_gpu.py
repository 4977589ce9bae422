"""Device-resident MLP training (GpuMLP: products through the tiled runtime,
elementwise steps in the K3-K7 kernels) against the reference's golden f64
trajectories and against the oracle at a larger width."""

from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import GpuMLP, Layer, Runtime, homogeneous_machine

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def relerr(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("act", ["sigmoid", "relu"])
@pytest.mark.parametrize("tile", [16, 4096])
def test_golden_trajectory(act, tile):
    g = np.load(G / "ann.npz")
    layers = [Layer(g[f"{act}_init_w{i}"], g[f"{act}_init_b{i}"], act, tag=f"layer{i}") for i in range(3)]
    mlp = GpuMLP(layers, machine=homogeneous_machine(2, gpus=[0, 0]), tile_size=tile)
    x = torch.as_tensor(g[f"{act}_x"], dtype=torch.float32).cuda()
    t = torch.as_tensor(g[f"{act}_t"], dtype=torch.float32).cuda()
    n, grads = mlp.loss_gradients(x, t)
    loss0 = float(mlp._loss.item()) / n
    assert abs(loss0 - g[f"{act}_loss0"][0]) <= 1e-5 * g[f"{act}_loss0"][0]
    for i, (gw, gb) in enumerate(grads):
        assert relerr(gw.cpu().numpy(), g[f"{act}_gw{i}"]) <= 1e-4
        assert relerr(gb.cpu().numpy(), g[f"{act}_gb{i}"]) <= 1e-4
    traj = np.array([mlp.train_step(x, t, 0.1) for _ in range(10)])
    ref = g[f"{act}_losses"]
    assert np.max(np.abs(traj - ref) / ref) <= 1e-5, (traj, ref)
    for i, (w, b) in enumerate(mlp.to_host()):
        assert relerr(w, g[f"{act}_final_w{i}"]) <= 1e-5
    assert mlp.products == 11 * 3 * 3  # 11 passes x 3 layers x (1 forward + 2 backward products)
    mlp.close()


def test_wide_net_against_blas_oracle():
    """784-2048-2048-2048-10, batch 2048 (cfg3 shape scaled by 1/4): three SGD
    steps on the GPU vs the float64 oracle with the same init (SURVEY §7 init)."""
    rng = np.random.default_rng(3)
    sizes = [784, 2048, 2048, 2048, 10]
    layers = [Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}")
              for i in range(4)]
    x, t = O.random_regression(rng, 2048, 784, 10)
    oracle_layers = [O.OracleLayer(L.weights.copy(), L.bias.copy(), L.activation) for L in layers]
    mlp = GpuMLP(layers, tile_size=1024)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    for step in range(3):
        lg = mlp.train_step(xd, td, 0.5)
        lo = O.train_step(oracle_layers, x, t, 0.5, matmul=O.blas_matmul)
        assert abs(lg - lo) <= 1e-5 * lo, (step, lg, lo)
    for (w, b), L in zip(mlp.to_host(), oracle_layers):
        assert relerr(w, L.weights) <= 1e-5 and relerr(b, L.bias) <= 1e-5
    mlp.close()


@pytest.mark.parametrize("capacity", [0, 40])
def test_wide_out_of_core_against_blas_oracle(capacity):
    """BASELINE cfg5's shape scaled by 1/32 (784-2048-2048-2048, batch 1024, T=256,
    weights drawn on the device by GpuMLP.random) with the tile cache bounded to
    40 tiles -- below the 144 weight tiles alone, so tiles are evicted and
    re-staged inside every step -- against the float64 oracle; the bounded run
    must also equal the unbounded one bit for bit (eviction changes where a
    tile comes from, never how a product is summed)."""
    sizes = [784, 2048, 2048, 2048]
    rt = Runtime(homogeneous_machine(1, capacity_tiles=capacity or None, dtype=np.float32), 256)
    mlp = GpuMLP.random(sizes, seed=11, runtime=rt)
    oracle_layers = [O.OracleLayer(w, b, "sigmoid") for w, b in mlp.to_host()]
    g = torch.Generator(device="cuda").manual_seed(12)
    xd = torch.rand((1024, sizes[0]), device="cuda", generator=g) * 2 - 1
    td = torch.rand((1024, sizes[-1]), device="cuda", generator=g) * 2 - 1
    x, t = xd.double().cpu().numpy(), td.double().cpu().numpy()
    losses = []
    for step in range(3):
        losses.append(mlp.train_step(xd, td, 0.5))
        lo = O.train_step(oracle_layers, x, t, 0.5, matmul=O.blas_matmul)
        assert abs(losses[-1] - lo) <= 1e-5 * lo, (step, losses[-1], lo)
    for (w, b), L in zip(mlp.to_host(), oracle_layers):
        assert relerr(w, L.weights) <= 1e-5 and relerr(b, L.bias) <= 1e-5
    _WIDE_RUNS[capacity] = (losses, mlp.to_host(), mlp.cache_counts["evictions"])
    if len(_WIDE_RUNS) == 2:  # the bounded run evicts far more and computes the same bits
        (l0, p0, e0), (l1, p1, e1) = _WIDE_RUNS[0], _WIDE_RUNS[40]
        assert e1 > 10 * max(e0, 1), (e0, e1)
        assert l0 == l1
        for (w0, b0), (w1, b1) in zip(p0, p1):
            assert np.array_equal(w0, w1) and np.array_equal(b0, b1)
    mlp.close()


_WIDE_RUNS: dict = {}


def test_stream_ordered_matches_blocking():
    """GpuMLP's stream-ordered products (no host wait between scheduling rounds)
    produce bit-identical trajectories and weights to blocking products."""
    rng = np.random.default_rng(5)
    sizes = [300, 700, 500, 7]
    base = [Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}")
            for i in range(3)]
    x, t = O.random_regression(rng, 333, 300, 7)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    runs = {}
    for ordered in (False, True):
        layers = [Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base]
        mlp = GpuMLP(layers, machine=homogeneous_machine(2, gpus=[0, 0]), tile_size=128, stream_ordered=ordered)
        losses = [mlp.train_step(xd, td, 0.2) for _ in range(4)]
        runs[ordered] = (losses, mlp.to_host())
        mlp.close()
    assert runs[True][0] == runs[False][0]
    for (w1, b1), (w0, b0) in zip(runs[True][1], runs[False][1]):
        assert np.array_equal(w1, w0) and np.array_equal(b1, b0)


def test_data_parallel_shards_sum_to_full_batch():
    """The data-parallel gradient: two half-batch shards with the MSE scaled by
    the global element count sum to the full-batch gradient (what the NCCL
    all-reduce forms across ranks), and a 1-rank NCCL group trains exactly like
    the plain model."""
    rng = np.random.default_rng(8)
    sizes = [200, 600, 300, 5]
    base = [Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}") for i in range(3)]
    x, t = O.random_regression(rng, 512, 200, 5)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()

    def grads(mlp, xs, ts, world):
        mlp.world = world  # the global count the MSE gradient is scaled by
        n, g = mlp.loss_gradients(xs, ts)
        return [(w.double().cpu(), b.double().cpu()) for w, b in g], float(mlp._loss.item())

    full = GpuMLP([Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base], tile_size=128)
    g_full, loss_full = grads(full, xd, td, 1)
    half = GpuMLP([Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base], tile_size=128)
    g0, l0 = grads(half, xd[:256], td[:256], 2)
    g1, l1 = grads(half, xd[256:], td[256:], 2)
    for (wf, bf), (w0, b0), (w1, b1) in zip(g_full, g0, g1):
        assert relerr((w0 + w1).numpy(), wf.numpy()) <= 1e-5 and relerr((b0 + b1).numpy(), bf.numpy()) <= 1e-5
    assert abs((l0 + l1) - loss_full) <= 1e-6 * loss_full
    full.close()
    half.close()

    import os

    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        runs = []
        for pg in (None, dist.group.WORLD):
            mlp = GpuMLP([Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base],
                         tile_size=128, process_group=pg)
            runs.append([mlp.train_step(xd, td, 0.2) for _ in range(3)])
            mlp.close()
        assert runs[0] == runs[1]
    finally:
        dist.destroy_process_group()


def test_write_through_matches_convert():
    """Producers writing the next round's operand tiles straight into the cache
    (cache_as) give bit-identical training to converting them on demand, and
    run fewer split/convert launches."""
    rng = np.random.default_rng(13)
    sizes = [256, 1024, 768, 512]
    base = [Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}") for i in range(3)]
    x, t = O.random_regression(rng, 512, 256, 512)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    runs = {}
    for wt in (False, True):
        mlp = GpuMLP([Layer(L.weights.copy(), L.bias.copy(), L.activation, tag=L.tag) for L in base],
                     tile_size=256, write_through=wt, stream_ordered=False)
        launches = []
        orig = mlp.rt.multiply_batch

        def counting(prods, _orig=orig):
            st = _orig(prods)
            launches.append(st.gpu_launches)
            return st

        mlp.rt.multiply_batch = counting
        losses = [mlp.train_step(xd, td, 0.2) for _ in range(3)]
        runs[wt] = (losses, mlp.to_host(), sum(launches))
        mlp.close()
    assert runs[True][0] == runs[False][0]
    for (w1, b1), (w0, b0) in zip(runs[True][1], runs[False][1]):
        assert np.array_equal(w1, w0) and np.array_equal(b1, b0)
    assert runs[True][2] < runs[False][2]


def test_async_steps_match_blocking():
    """train_step_async (loss read after the next step is enqueued) computes the
    same trajectory as train_step, bit for bit."""
    sizes = [784, 512, 512, 10]
    runs = []
    for use_async in (False, True):
        mlp = GpuMLP.random(sizes, seed=21, runtime=Runtime(homogeneous_machine(1, dtype=np.float32), 256))
        g = torch.Generator(device="cuda").manual_seed(22)
        x = torch.rand((512, 784), device="cuda", generator=g)
        t = torch.rand((512, 10), device="cuda", generator=g)
        if use_async:
            pend = [mlp.train_step_async(x, t, 0.3) for _ in range(6)]
            losses = [p.result() for p in pend]
        else:
            losses = [mlp.train_step(x, t, 0.3) for _ in range(6)]
        runs.append((losses, mlp.to_host()))
        mlp.close()
    assert runs[0][0] == runs[1][0]
    for (w0, b0), (w1, b1) in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(w0, w1) and np.array_equal(b0, b1)


def test_fused_sgd_matches_gradient_buffers():
    """The fused update (dW products accumulating straight into W) trains like
    the dW-buffer + SGD-kernel path, to fp32 rounding."""
    sizes = [784, 1024, 1024, 10]
    runs = []
    for fused in (True, False):
        mlp = GpuMLP.random(sizes, seed=31, runtime=Runtime(homogeneous_machine(1, dtype=np.float32), 512),
                            fused_sgd=fused)
        g = torch.Generator(device="cuda").manual_seed(32)
        x = torch.rand((1024, 784), device="cuda", generator=g) * 2 - 1
        t = torch.rand((1024, 10), device="cuda", generator=g) * 2 - 1
        runs.append(([mlp.train_step(x, t, 0.5) for _ in range(4)], mlp.to_host()))
        mlp.close()
    (l0, p0), (l1, p1) = runs
    assert np.allclose(l0, l1, rtol=1e-6, atol=0)
    for (w0, b0), (w1, b1) in zip(p0, p1):
        assert relerr(w0, w1) <= 1e-6 and np.array_equal(b0, b1)


@pytest.mark.parametrize("fused", [True, False])
def test_skip_input_grad_same_trajectory(fused):
    """skip_input_grad drops the first layer's dX product (ann.py:171-172 computes
    it; nothing reads it): same losses and weights, one product fewer per step."""
    sizes = [300, 256, 200, 10]
    rng = np.random.default_rng(41)
    layers = [Layer.random(sizes[i], sizes[i + 1], rng, activation="sigmoid", scale=1.0 / np.sqrt(sizes[i]),
                           tag=f"layer{i}") for i in range(3)]
    x = torch.as_tensor(rng.uniform(-1, 1, (512, sizes[0])), dtype=torch.float32).cuda()
    t = torch.as_tensor(rng.uniform(-1, 1, (512, sizes[-1])), dtype=torch.float32).cuda()
    runs = {}
    for skip in (False, True):
        mlp = GpuMLP(layers, machine=homogeneous_machine(1, dtype=np.float32), tile_size=128, fused_sgd=fused,
                     skip_input_grad=skip)
        losses = [mlp.train_step(x, t, 0.1) for _ in range(4)]
        runs[skip] = (losses, mlp.to_host(), mlp.products)
        mlp.close()
    # the other products are unchanged; only their grouping into launches may differ
    assert np.allclose(runs[False][0], runs[True][0], rtol=1e-6, atol=0)
    for (w0, b0), (w1, b1) in zip(runs[False][1], runs[True][1]):
        assert relerr(w1, w0) <= 1e-6 and relerr(b1, b0) <= 1e-6
    assert runs[False][2] - runs[True][2] == 4  # one dX product per step


def test_cfg3_full_shape_losses_vs_f64_oracle():
    """BASELINE cfg3 at its full shape, 784-8192-8192-8192-10 x 8192 (SURVEY §8d
    init: per-layer scale 1/sqrt(fan_in), random_regression data): 3 SGD steps
    on the GPU in both precisions against the reference's train_step algebra in
    float64 (oracle.train_step with BLAS products, ann.py:239-248); per-step loss
    relative error <= 1e-5 (fp32acc) / 1e-2 (bf16)."""
    sizes, batch = [784, 8192, 8192, 8192, 10], 8192
    rng = np.random.default_rng(0)
    layers = [Layer.random(sizes[i], sizes[i + 1], rng, activation="sigmoid", scale=1.0 / np.sqrt(sizes[i]),
                           tag=f"layer{i}") for i in range(4)]
    x = rng.uniform(-1.0, 1.0, size=(batch, sizes[0]))
    t = rng.uniform(-1.0, 1.0, size=(batch, sizes[-1]))
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    got = {}
    for precision in ("fp32acc", "bf16"):
        mlp = GpuMLP(layers, machine=homogeneous_machine(1, dtype=np.float32), tile_size=4096, precision=precision)
        got[precision] = [mlp.train_step(xd, td, 0.1) for _ in range(3)]
        mlp.close()
    ol = [O.OracleLayer(np.array(L.weights, np.float64), np.array(L.bias, np.float64), "sigmoid") for L in layers]
    ref = [O.train_step(ol, x, t, 0.1, matmul=O.blas_matmul) for _ in range(3)]
    for precision, tol in (("fp32acc", 1e-5), ("bf16", 1e-2)):
        errs = [abs(g - r) / abs(r) for g, r in zip(got[precision], ref)]
        assert max(errs) <= tol, (precision, errs)


@pytest.mark.parametrize("m,k,n,tile", [(8192, 4096, 8192, 4096),   # full tiles: fused into K1's epilogue
                                        (1000, 4096, 768, 256),     # ragged rows, split-K launches: tile passes
                                        (512, 10, 640, 256),        # k = 10: CUDA-core tasks
                                        (4096, 2048, 10, 4096)])    # 10 wide: transposed tensor-core product
def test_fused_colsum_block_sums(m, k, n, tile):
    """tr_product.colsum: the 32-row block column sums of the FINAL output (after
    the act_grad post-op), whichever kernel path each task takes; summed by
    tr_mlp_colsum_finish they are db = colsum(dY) (ann.py:173)."""
    from paper_1511_04348_b200 import _native as N

    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(k, n, device="cuda", generator=g)
    act = torch.rand(m, n, device="cuda", generator=g)
    out = torch.empty(m, n, device="cuda")
    parts = torch.full((-(-m // 32), n), float("nan"), device="cuda")
    with Runtime(homogeneous_machine(1, dtype=np.float32), tile) as rt:
        rt.multiply_batch([dict(a=a, b=b, out=out, post=("act_grad", act, "sigmoid"), colsum=parts)])
    torch.cuda.synchronize()
    ref = torch.nn.functional.pad(out.double(), (0, 0, 0, parts.shape[0] * 32 - m)).view(-1, 32, n).sum(1)
    assert not torch.isnan(parts).any()
    assert float(torch.linalg.norm(parts.double() - ref) / torch.linalg.norm(ref)) <= 1e-6
    db = torch.empty(n, device="cuda")
    N.call("tr_mlp_colsum_finish", parts.data_ptr(), parts.shape[0], n, db.data_ptr(), None)
    torch.cuda.synchronize()
    want = out.double().sum(0)
    assert float(torch.linalg.norm(db.double() - want) / torch.linalg.norm(want)) <= 1e-6


def test_fused_colsum_same_trajectory_as_colsum_pass():
    sizes = [300, 512, 256, 10]
    rng = np.random.default_rng(43)
    layers = [Layer.random(sizes[i], sizes[i + 1], rng, activation="sigmoid", scale=1.0 / np.sqrt(sizes[i]),
                           tag=f"layer{i}") for i in range(3)]
    x = torch.as_tensor(rng.uniform(-1, 1, (1024, sizes[0])), dtype=torch.float32).cuda()
    t = torch.as_tensor(rng.uniform(-1, 1, (1024, sizes[-1])), dtype=torch.float32).cuda()
    runs = {}
    for fused in (False, True):
        mlp = GpuMLP(layers, machine=homogeneous_machine(1, dtype=np.float32), tile_size=256, fused_colsum=fused)
        runs[fused] = ([mlp.train_step(x, t, 0.1) for _ in range(4)], mlp.to_host())
        mlp.close()
    assert np.allclose(runs[False][0], runs[True][0], rtol=1e-6, atol=0)
    for (w0, b0), (w1, b1) in zip(runs[False][1], runs[True][1]):
        assert relerr(w1, w0) <= 1e-6 and relerr(b1, b0) <= 1e-6


def test_tile_parallel_mlp_on_green_context_devices():
    """cfg5's machine in miniature: the MLP's products shared tile by tile (the
    reference's TiledBackend semantics, ann.py:78-104) by three green-context
    devices, one throttled; 5 SGD steps against the float64 oracle, and every
    device did part of the work."""
    from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix

    sizes = [256, 1024, 768, 10]
    rng = np.random.default_rng(47)
    layers = [Layer.random(sizes[i], sizes[i + 1], rng, activation="sigmoid", scale=1.0 / np.sqrt(sizes[i]),
                           tag=f"layer{i}") for i in range(3)]
    x, t = O.random_regression(rng, 512, sizes[0], sizes[-1])
    m = Machine([DeviceSpec(0, gpu=0, sms=16), DeviceSpec(1, gpu=0, sms=16), DeviceSpec(2, gpu=0, sms=8, slots=2)],
                ProximityMatrix.uniform(3), dtype=np.float32)
    mlp = GpuMLP(layers, machine=m, tile_size=128)
    xd = torch.as_tensor(x, dtype=torch.float32).cuda()
    td = torch.as_tensor(t, dtype=torch.float32).cuda()
    got = [mlp.train_step(xd, td, 0.1) for _ in range(5)]
    assert all(v > 0 for v in mlp.device_macs), mlp.device_macs
    mlp.close()
    ol = [O.OracleLayer(np.array(L.weights, np.float64), np.array(L.bias, np.float64), "sigmoid") for L in layers]
    ref = [O.train_step(ol, x, t, 0.1, matmul=O.blas_matmul) for _ in range(5)]
    assert max(abs(g - r) / r for g, r in zip(got, ref)) <= 1e-5, (got, ref)
