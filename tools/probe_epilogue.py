"""Probe: tile_gemm epilogue cost by variant (8192^3 fp32acc products on device
tensors, T=4096): plain, transposed B, act_grad post, bias_act post, write-through.
Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 8192, 4096
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g)
b = torch.randn(n, n, device="cuda", generator=g)
aux = torch.rand(n, n, device="cuda", generator=g)
bias = torch.randn(n, device="cuda", generator=g)
c = torch.empty(n, n, device="cuda")
rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T)
variants = {
    "plain": dict(),
    "transpose_a": dict(transpose_a=True),
    "transpose_b": dict(transpose_b=True),
    "act_grad": dict(post=("act_grad", aux, "sigmoid")),
    "bias_act": dict(post=("bias_act", bias, "sigmoid")),
    "tb+act_grad": dict(transpose_b=True, post=("act_grad", aux, "sigmoid")),
    "write_through": dict(cache_as="WT"),
    "bias_act+wt": dict(post=("bias_act", bias, "sigmoid"), cache_as="WT"),
    "tb+act_grad+wt": dict(transpose_b=True, post=("act_grad", aux, "sigmoid"), cache_as="WT"),
    "ta+axpy": dict(transpose_a=True, axpy=-0.01),
    "ta+axpy+wt": dict(transpose_a=True, axpy=-0.01, cache_as="WT"),
    "axpy": dict(axpy=-0.01),
}
for name, kw in variants.items():
    ts = []
    for i in range(6):
        p = dict(a=a, b=b, out=c, a_uid="A", b_uid="B", **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rt.multiply_batch([p])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        rt.forget("WT")
    t = float(np.median(ts[2:]))
    print(f"{name:16s} {t:8.3f} ms  {2 * n ** 3 / t / 1e9:7.1f} TF/s", flush=True)
