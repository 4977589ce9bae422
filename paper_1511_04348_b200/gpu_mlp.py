"""Device-resident MLP training through the tiled GPU runtime (BASELINE cfg3).

Same algebra and the same 3·L products per step as the reference's
``train_step`` (ann.py:239-248, Eqs. 1-4 of the paper):

    forward   Y_l = X_l W_l (product) ; Y_l += b_l ; X_{l+1} = act(Y_l)   (K3)
    loss      dOut = 2 (pred - target) / size ; loss = mean (pred - target)^2 (K4b)
    backward  dY_l = dOut * act'(Y_l, X_{l+1})                             (K4)
              dW_l = X_l^T dY_l        (product, transposed A: layout, no copy)
              dX_l = dY_l W_l^T        (product, transposed B; also for l = 0,
                                        as the reference does)
              db_l = colsum dY_l   (K5; for l < L-1 summed from the 32-row block
                                    sums the dX product's epilogue emits with dY_l)
    update    W_l -= lr dW_l ; b_l -= lr db_l ; version += 1               (K6)

Every product is ``Runtime.multiply`` on device-resident operands: tiles are
admitted into the HBM tile cache by uid (activation/gradient uids are fresh
per step, weight uids are versioned exactly like ``Layer.weight_uid``), so the
backward products hit the tiles the forward products cached.  Activations and
parameters are float32 on the device; the products run in the FP32-accurate
mode; the loss is accumulated in float64.

Data parallel over a ``torch.distributed`` process group (one process per GPU,
NCCL): each rank trains on its shard of the global batch, the MSE gradient is
scaled by the GLOBAL element count, and each layer's (dW, db) is all-reduced
(sum) as soon as its backward round is enqueued -- on NCCL's stream, so the
exchange overlaps the remaining backward products -- before the SGD update.
The sum of the shards' gradients is the full-batch gradient of the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .devices import Machine, homogeneous_machine
from .scheduler import Runtime

_ACT = {"identity": N.TR_ACT_IDENTITY, "sigmoid": N.TR_ACT_SIGMOID, "relu": N.TR_ACT_RELU}


def _ptr(t) -> int:
    return t.data_ptr()


@dataclass
class DeviceLayer:
    w: object  # torch.Tensor fan_in x fan_out (float32, cuda)
    b: object | None
    activation: str
    tag: str
    version: int = 0

    @property
    def weight_uid(self) -> str:
        return f"{self.tag}.w.v{self.version}"


class PendingLoss:
    """The loss of an enqueued training step: ``result()`` waits for its D2H copy."""

    def __init__(self, host, event, n):
        self._host, self._event, self._n = host, event, n

    def result(self) -> float:
        self._event.synchronize()
        return float(self._host[0]) / self._n


class GpuMLP:
    """A float32 MLP living in HBM, trained through a tiled ``Runtime`` session."""

    def __init__(self, layers, machine: Machine | None = None, tile_size: int = 4096, precision: str = "fp32acc",
                 device: int = 0, runtime: Runtime | None = None, stream_ordered: bool = True,
                 process_group=None, write_through: bool = True, fused_sgd: bool = True,
                 write_through_weights: bool | None = None, skip_input_grad: bool = False,
                 fused_colsum: bool = True):
        import torch

        if precision == "exact" or (runtime is not None and runtime.precision == "exact"):
            raise ValueError("GpuMLP fuses bias/activation/SGD into the tile GEMMs; precision 'exact' "
                             "covers plain products only (use 'fp32acc')")
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.layers: list[DeviceLayer] = []
        for i, L in enumerate(layers):
            if isinstance(L, DeviceLayer):  # already in HBM (GpuMLP.random): taken as is
                self.layers.append(L)
                continue
            w = torch.as_tensor(np.asarray(L.weights), dtype=torch.float32).to(self.dev).contiguous()
            b = None if L.bias is None else torch.as_tensor(np.asarray(L.bias), dtype=torch.float32).to(self.dev)
            self.layers.append(DeviceLayer(w, b, L.activation, getattr(L, "tag", f"layer{i}")))
        if runtime is None:
            machine = machine or homogeneous_machine(1, dtype=np.float32, gpus=[device])
            runtime = Runtime(machine, tile_size, precision=precision)
        self.rt = runtime
        self.stream_ordered = stream_ordered
        self.write_through = write_through  # producers write the next round's operand tiles into the cache
        self.fused_sgd = fused_sgd  # one process: dW products accumulate straight into W (no gradient buffer)
        # fused SGD: the update product also writes the new weights' tiles into the cache
        self.write_through_weights = write_through if write_through_weights is None else write_through_weights
        # ann.py:171-172 computes dX of the first layer too, though nothing reads it;
        # True skips that product (cfg3: 784-wide output, ~1.5 % of a step's flops)
        self.skip_input_grad = skip_input_grad
        # db = colsum(dY) from the dX product's epilogue (32-row block sums) instead of a pass over dY
        self.fused_colsum = fused_colsum
        self.pg = process_group
        if process_group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
        else:
            self.world = 1
        self._pending = []  # in-flight gradient all-reduces of the current step
        self._loss = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self._bufs: dict = {}
        self.products = 0
        # tile-cache counters summed over every product (directory bookkeeping, exact
        # at enqueue even when the products run stream-ordered)
        self.cache_counts = dict.fromkeys(("l1_hits", "host_fetches", "evictions", "writebacks"), 0)
        # per logical device: tasks and rows x cols x K of the products it ran (work shares)
        n_dev = self.rt.machine.n_devices
        self.device_tasks = [0] * n_dev
        self.device_macs = [0] * n_dev

    @classmethod
    def random(cls, sizes, activation: str = "sigmoid", seed: int = 0, device: int = 0, **kw) -> "GpuMLP":
        """Layers initialised in HBM: uniform(-1/sqrt(fan_in), 1/sqrt(fan_in)) weights
        then bias per layer, as ``Layer.random`` with the per-layer scale (SURVEY
        §8d), drawn by a seeded device generator -- for widths (BASELINE cfg5,
        65536) whose host-side f64 initialisation would take minutes."""
        import torch

        dev = torch.device("cuda", device)
        g = torch.Generator(device=dev).manual_seed(seed)
        layers = []
        for i in range(len(sizes) - 1):
            s = 1.0 / float(np.sqrt(sizes[i]))
            w = torch.empty((sizes[i], sizes[i + 1]), dtype=torch.float32, device=dev).uniform_(-s, s, generator=g)
            b = torch.empty(sizes[i + 1], dtype=torch.float32, device=dev).uniform_(-s, s, generator=g)
            layers.append(DeviceLayer(w, b, activation, f"layer{i}"))
        return cls(layers, device=device, **kw)

    # -- helpers -----------------------------------------------------------
    def _buf(self, name, shape):
        t = self._bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape):
            t = self.torch.empty(shape, dtype=self.torch.float32, device=self.dev)
            self._bufs[name] = t
        return t

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def _batch(self, prods):
        """Run independent products as one scheduling round (fused epilogues allowed).

        Stream-ordered (tr_session_set_async): every operand lives in HBM, so the
        call returns once the tasks are enqueued and the torch stream waits for
        them; the host prepares the next round while this one runs.
        """
        self.rt.set_stream(self._stream(), ordered=self.stream_ordered)
        try:
            st = self.rt.multiply_batch(prods)
            for k in self.cache_counts:
                self.cache_counts[k] += getattr(st.cache, k)
            for d, ds in st.devices.items():
                self.device_tasks[d] += ds.tasks_completed
                self.device_macs[d] += ds.macs
        finally:
            self.rt.set_stream(self._stream(), ordered=False)
        self.products += len(prods)

    # -- one pass ------------------------------------------------------------
    def _allreduce(self, *tensors):
        """Sum over the data-parallel group, asynchronously (NCCL's stream waits
        for the current stream, so the products that made the tensors are done)."""
        if self.pg is None or self.world == 1:
            return
        import torch.distributed as dist

        for t in tensors:
            if t is not None:
                self._pending.append(dist.all_reduce(t, group=self.pg, async_op=True))

    def loss_gradients(self, x, target, lr: float | None = None):
        """Forward + backward without update; returns (n, [(dW, db)]) with the loss
        sum left in ``self._loss`` (device).

        Fusion: the forward products write act(X W + b) directly (the epilogue
        applies bias and activation; only the activation output is kept, which
        is all act'() needs); the backward dX product of layer l multiplies by
        act'(A_{l-1}) in its epilogue, producing dY_{l-1} directly; dW_l and
        dX_l are independent and share one scheduling round.

        With ``lr`` (the fused SGD step, one process): no dW is materialised --
        the dW_l product accumulates straight into the weights, W_l += (-lr)
        X_l^T dY_l (an axpy product), one round later, next to dX_{l-1}, so it
        runs after dX_l has read W_l; the returned dW entries are None.
        """
        s = self._stream()
        xs, uids = [], []
        cur, cur_uid = x, self.rt.fresh_uid("x")
        for li, L in enumerate(self.layers):
            xs.append(cur)
            uids.append(cur_uid)
            a = self._buf(f"a{li}", (cur.shape[0], L.w.shape[1]))
            nxt = self.rt.fresh_uid("x")
            # the activation is the next product's A: its tiles enter the cache as they are produced
            self._batch([dict(a=cur, b=L.w, out=a, a_uid=cur_uid, b_uid=L.weight_uid,
                              post=("bias_act", L.b, L.activation), cache_as=nxt if self.write_through else None)])
            cur, cur_uid = a, nxt
        self._step_uids = list(uids) + [cur_uid]
        pred = cur
        d_out = self._buf("dout", pred.shape)
        N.call("tr_mlp_mse_grad_global", _ptr(d_out), _ptr(pred), _ptr(target), pred.numel(),
               pred.numel() * self.world, _ptr(self._loss), s)
        last = len(self.layers) - 1
        d_y = self._buf(f"dy{last}", pred.shape)
        N.call("tr_mlp_act_grad", _ptr(d_y), _ptr(d_out), None, _ptr(pred), d_y.numel(),
               _ACT[self.layers[last].activation], s)
        grads = [None] * len(self.layers)
        dy_uid = self.rt.fresh_uid("dy")
        update = None  # fused SGD: the layer above's W += (-lr) X^T dY, run with this layer's round
        cs_parts = None  # block column sums of the current dY (fused into the producing product)
        for li in range(last, -1, -1):
            L = self.layers[li]
            self._step_uids.append(dy_uid)
            next_dy = self.rt.fresh_uid("dy")
            d_x = self._buf(f"dy{li - 1}" if li > 0 else "dx0", xs[li].shape)
            dx = dict(a=d_y, b=L.w, out=d_x, transpose_b=True, a_uid=dy_uid, b_uid=L.weight_uid)
            if li > 0:  # dX_l * act'(A_{l-1}) = dY_{l-1}  (xs[li] is A_{l-1})
                dx["post"] = ("act_grad", xs[li], self.layers[li - 1].activation)
                if self.write_through:
                    dx["cache_as"] = next_dy  # dY_{l-1} is the next round's operand
                if self.fused_colsum and self.layers[li - 1].b is not None and self.rt.tile_size % 32 == 0:
                    # db_{l-1} = colsum(dY_{l-1}): block sums from the producing epilogue
                    dx["colsum"] = self._buf(f"cs{li - 1}", (-(-d_x.shape[0] // 32), d_x.shape[1]))
            dw = dict(a=xs[li], b=d_y, transpose_a=True, a_uid=uids[li], b_uid=dy_uid)
            dxs = [] if (li == 0 and self.skip_input_grad) else [dx]
            if lr is None:
                d_w = dw["out"] = self._buf(f"dw{li}", L.w.shape)
                self._batch([dw] + dxs)
            else:
                d_w = None
                dw.update(out=L.w, axpy=-float(lr))
                if self.write_through_weights:  # the updated weights' tiles enter the cache as the next version
                    dw["cache_as"] = f"{L.tag}.w.v{L.version + 1}"
                if dxs or update:
                    self._batch(dxs + ([update] if update else []))
                update = dw
            d_b = None
            if L.b is not None:
                d_b = self._buf(f"db{li}", L.b.shape)
                if cs_parts is not None:  # the block sums came with dY (fused colsum)
                    N.call("tr_mlp_colsum_finish", _ptr(cs_parts), cs_parts.shape[0], cs_parts.shape[1], _ptr(d_b), s)
                else:
                    N.call("tr_mlp_colsum", _ptr(d_y), d_y.shape[0], d_y.shape[1], _ptr(d_b), s)
            self._allreduce(d_w, d_b)  # overlaps the next (lower) layer's backward round
            grads[li] = (d_w, d_b)
            d_y, dy_uid = d_x, next_dy
            cs_parts = dx.get("colsum")
        if update:
            self._batch([update])
        return pred.numel(), grads

    def train_step(self, x, target, lr: float) -> float:
        """One SGD step (ann.py:239-248); returns the MSE loss (read back to the host)."""
        return self.train_step_async(x, target, lr).result()

    def train_step_async(self, x, target, lr: float) -> "PendingLoss":
        """``train_step`` without the host wait: the step is enqueued, its loss is
        copied to pinned host memory in stream order, and ``.result()`` waits for
        that copy only -- so the host prepares step i+1 while step i runs."""
        fused = self.fused_sgd and self.world == 1  # data parallel: all-reduce dW first
        n, grads = self.loss_gradients(x, target, lr if fused else None)
        for h in self._pending:  # the current stream waits for every gradient all-reduce
            h.wait()
        self._pending = []
        self._allreduce(self._loss)
        for h in self._pending:
            h.wait()
        self._pending = []
        n *= self.world
        s = self._stream()
        for L, (d_w, d_b) in zip(self.layers, grads):
            if d_w is not None:
                N.call("tr_mlp_sgd", _ptr(L.w), _ptr(d_w), L.w.numel(), float(lr), s)
            if L.b is not None:
                N.call("tr_mlp_sgd", _ptr(L.b), _ptr(d_b), L.b.numel(), float(lr), s)
            self.rt.forget(L.weight_uid)  # this version is dead after the update
            L.version += 1
        for uid in self._step_uids:  # this step's activations and gradients are dead too
            self.rt.forget(uid)
        host = self.torch.empty(1, dtype=self.torch.float64, pin_memory=True)  # torch's cached pinned pool
        host.copy_(self._loss, non_blocking=True)
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream(self.dev))
        return PendingLoss(host, ev, n)

    def to_host(self):
        """[(W, b)] as float64 numpy arrays."""
        return [(L.w.double().cpu().numpy(), None if L.b is None else L.b.double().cpu().numpy())
                for L in self.layers]

    def close(self):
        self.rt.close()
