"""MC-MLP training (BASELINE config 3) on the MCF operators.

The reference composes this from its library: MCSequential of MCLinear layers
(nn.hpp:49-92, 162-201) with ReLU (autodiff.hpp:133-144), cross-entropy
(autodiff.hpp:541-582), reverse-mode tape (autodiff.hpp:209-228) and MC-SGD
applied through Grow-ExpN (optim.hpp:54-77, mc_ops.hpp:509-513).  Here one
training step is a fixed sequence of C-ABI calls on feature-major activations
(features x batch):

  forward   Z = W . A_prev (MC x Tensor, mcf_bmm_mcn, plan FAST or reference
            order), h = approx(add_mcn(Z, b)), A = relu(h)   (mcf_mlp_bias_act)
  loss      mcf_mlp_cross_entropy (terms, gradient / N_global, ordered sum)
  backward  dW = G A_prev^T, dA = approx(W)^T G masked by h_prev > 0,
            db = row sums of G  (reference-order plan: ordered binary32,
            mcf_gemm_f32_ordered / mcf_rowsum_f32_ordered -- matmul2d
            semantics; plan FAST: mcf_gemm_f32_fast / mcf_rowsum_f32_fast)
  exchange  data parallel: one flat binary32 gradient buffer, all_reduce(sum)
            over the process group (NCCL over NVLink on GPUs)
  update    mcf_sgd_grow: w <- grow_expn(w, -lr * g), identical on every rank

Single process with the reference-order plan, every step is bit-identical to
the reference's own training loop (tests/test_gpu_mlp.py); with plan FAST the
forward MC products run on the INT8 tensor-core splitting (the FP64 pipe for
short layers), the backward on FP32 library GEMMs, and the loss trajectory
stays within the reference's rounding spread.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import B32, FAST, FAST_FP64, SEQUENTIAL, _check, lib
from . import data as _data


def init_params(dims, nc=2, seed=3000):
    """Kaiming-uniform fan-in init (nn.hpp:41-47, 55-59): per layer the weight
    draws U(-1/sqrt(in), 1/sqrt(in)) then the bias draws, one Rng stream; each
    binary64 draw split into nc binary32 components (BASELINE config 3)."""
    counts = [dims[l + 1] * dims[l] + dims[l + 1] for l in range(len(dims) - 1)]
    u = _data.uniform(seed, sum(counts))
    params, off = [], 0
    for l in range(len(dims) - 1):
        fan_in, out = dims[l], dims[l + 1]
        bound = 1.0 / np.sqrt(float(fan_in))
        w = -bound + 2.0 * bound * u[off:off + out * fan_in]
        off += out * fan_in
        b = -bound + 2.0 * bound * u[off:off + out]
        off += out
        params.append((_data.split(w, nc).reshape(out, fan_in, nc), _data.split(b, nc).reshape(out, nc)))
    return params


def make_batch(n, in_dim=784, classes=10, seed_x=3001, seed_y=3002):
    """X ~ N(0,1) rounded to binary32 (Rng::normal), labels Rng::below(classes)."""
    x = _data.normal(seed_x, n * in_dim).astype(np.float32).reshape(n, in_dim)
    y = _data.below(seed_y, classes, n).astype(np.int32)
    return x, y


class GradExchange:
    """Flat binary32 gradient buffer + sum all-reduce across a process group.
    Works for any torch device/backend (NCCL on B200s, gloo on CPU tests).

    Buckets: reduce_bucket(b) starts an asynchronous all-reduce of a
    contiguous run of views as soon as the backward pass has written them
    (one layer's dW and db), so the exchange of layer l overlaps the
    backward GEMMs of layer l-1; finish() waits for every bucket
    (and reduces the loss sum).  all_reduce() is the one-shot form."""

    def __init__(self, shapes, device, group=None):
        self.shapes = shapes
        sizes = [int(np.prod(s)) for s in shapes]
        self.flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        self.views, self.offsets, off = [], [], 0
        for s, n in zip(shapes, sizes):
            self.views.append(self.flat[off:off + n].view(*s))
            self.offsets.append((off, off + n))
            off += n
        self.group = group
        self._pending = []

    def reduce_bucket(self, first_view: int, last_view: int):
        """Start the sum all-reduce of views first_view..last_view (inclusive)."""
        if self.world() <= 1:
            return
        import torch.distributed as dist

        a, b = self.offsets[first_view][0], self.offsets[last_view][1]
        self._pending.append(dist.all_reduce(self.flat[a:b], op=dist.ReduceOp.SUM, group=self.group,
                                             async_op=True))

    def finish(self, loss_sum: torch.Tensor = None):
        """Wait for the started buckets; reduce the loss sum."""
        for h in self._pending:
            h.wait()
        self._pending = []
        if self.world() > 1 and loss_sum is not None:
            import torch.distributed as dist

            dist.all_reduce(loss_sum, op=dist.ReduceOp.SUM, group=self.group)

    def world(self):
        if self.group is None:
            return 1
        import torch.distributed as dist

        return dist.get_world_size(self.group)

    def all_reduce(self, loss_sum: torch.Tensor = None):
        if self.world() > 1:
            import torch.distributed as dist

            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
            if loss_sum is not None:
                dist.all_reduce(loss_sum, op=dist.ReduceOp.SUM, group=self.group)


class MCMLP:
    """Device-resident MC-MLP; `step()` runs forward, loss, backward, gradient
    exchange and the MC-SGD update, and returns the step's loss."""

    def __init__(self, dims, params, lr=0.01, nc=2, plan=FAST, group=None, device="cuda"):
        self.dims, self.nc, self.lr, self.plan = list(dims), nc, float(lr), plan
        self.L = len(dims) - 1
        self.W = [torch.from_numpy(np.ascontiguousarray(w)).to(device) for w, _ in params]
        self.b = [torch.from_numpy(np.ascontiguousarray(b)).to(device) for _, b in params]
        shapes = []
        for l in range(self.L):
            shapes += [(dims[l + 1], dims[l]), (dims[l + 1],)]
        self.grads = GradExchange(shapes, device, group)
        self.lib = lib()
        self._bufs = None

    def _alloc(self, n):
        if self._bufs is not None and self._bufs["n"] == n:
            return self._bufs
        dev = self.W[0].device
        f = dict(dtype=torch.float32, device=dev)
        bufs = {"n": n}
        bufs["Z"] = [torch.empty((self.dims[l + 1], n, self.nc), **f) for l in range(self.L)]
        bufs["H"] = [torch.empty((self.dims[l + 1], n), **f) for l in range(self.L)]
        bufs["A"] = [torch.empty((self.dims[l + 1], n), **f) for l in range(self.L - 1)]
        bufs["G"] = [torch.empty((self.dims[l + 1], n), **f) for l in range(self.L)]
        bufs["Wa"] = [torch.empty((self.dims[l + 1], self.dims[l]), **f) for l in range(self.L)]
        bufs["terms"] = torch.empty(n, **f)
        bufs["loss"] = torch.zeros(1, **f)
        self._bufs = bufs
        return bufs

    def step(self, xt: torch.Tensor, labels: torch.Tensor, n_global: int) -> torch.Tensor:
        """xt: (in, n_local) binary32 (feature-major batch shard); labels (n_local,)
        int32.  Returns the (globally summed) loss terms as a 1-element device
        tensor, no host sync; loss_value() turns it into the loss."""
        L, nc, lib_ = self.L, self.nc, self.lib
        n = xt.shape[1]
        B = self._alloc(n)
        s = torch.cuda.current_stream().cuda_stream
        acts = [xt]
        for l in range(L):
            out_dim, in_dim = self.dims[l + 1], self.dims[l]
            last = l == L - 1
            _check(lib_.mcf_mlp_linear_fwd(self.W[l].data_ptr(), nc, acts[l].data_ptr(), out_dim, in_dim, n,
                                           self.b[l].data_ptr(), 0 if last else 1, B["Z"][l].data_ptr(),
                                           B["H"][l].data_ptr(), None if last else B["A"][l].data_ptr(), self.plan,
                                           s))
            if not last:
                acts.append(B["A"][l])
        # loss + dL/dlogits.  Plan FAST: the loss's sequential sum (8192
        # dependent additions) runs on a side stream, joined before the
        # gradient exchange, instead of delaying the backward
        fast = self.plan in (FAST, FAST_FP64)
        _check(lib_.mcf_mlp_cross_entropy(B["H"][L - 1].data_ptr(), labels.data_ptr(), self.dims[-1], n, n_global,
                                          B["G"][L - 1].data_ptr(), B["terms"].data_ptr(),
                                          None if fast else B["loss"].data_ptr(), s))
        loss_done = None
        if fast:
            cur = torch.cuda.current_stream()
            if getattr(self, "_loss_stream", None) is None:
                self._loss_stream = torch.cuda.Stream()
            side = self._loss_stream
            side.wait_stream(cur)
            _check(lib_.mcf_mlp_loss_sum(B["terms"].data_ptr(), n, B["loss"].data_ptr(), side.cuda_stream))
            loss_done = torch.cuda.Event()
            loss_done.record(side)
        # backward: the reference-order plan reproduces matmul2d's rounding
        # sequence; plan FAST uses FP32 library GEMMs and tree row sums
        gemm = lib_.mcf_gemm_f32_fast if fast else lib_.mcf_gemm_f32_ordered
        rowsum = lib_.mcf_rowsum_f32_fast if fast else lib_.mcf_rowsum_f32_ordered
        gv = self.grads.views
        # plan FAST: a layer's weight / bias gradients (and their all-reduce
        # bucket) run on a side stream while the main stream computes the
        # gradient for the layer below (dW and dA only share G)
        cur = torch.cuda.current_stream()
        wside = None
        if fast:
            if getattr(self, "_grad_stream", None) is None:
                self._grad_stream = torch.cuda.Stream()
            wside = self._grad_stream
        for l in range(L - 1, -1, -1):
            out_dim, in_dim = self.dims[l + 1], self.dims[l]
            G = B["G"][l]
            ws = s
            if wside is not None:
                wside.wait_stream(cur)  # G (and the activations) are ready
                ws = wside.cuda_stream
            # dW (out x in) = G (out x n) . A_prev^T  (A_prev is in x n)
            _check(gemm(0, 1, G.data_ptr(), n, acts[l].data_ptr(), n, gv[2 * l].data_ptr(), in_dim, out_dim, in_dim, n,
                        None, ws))
            _check(rowsum(G.data_ptr(), out_dim, n, gv[2 * l + 1].data_ptr(), ws))
            if wside is not None:
                with torch.cuda.stream(wside):
                    self.grads.reduce_bucket(2 * l, 2 * l + 1)  # overlaps the next layer's backward
            else:
                self.grads.reduce_bucket(2 * l, 2 * l + 1)  # overlaps the next layer's backward
            if l > 0:
                _check(lib_.mcf_approx(B32, self.W[l].data_ptr(), nc, B["Wa"][l].data_ptr(), out_dim * in_dim, s))
                # dA_prev (in x n) = approx(W)^T (in x out) . G (out x n), ReLU mask = H_{l-1}
                _check(gemm(1, 0, B["Wa"][l].data_ptr(), in_dim, G.data_ptr(), n, B["G"][l - 1].data_ptr(), n, in_dim,
                            n, out_dim, B["H"][l - 1].data_ptr(), s))
        if wside is not None:
            cur.wait_stream(wside)
        if loss_done is not None:
            torch.cuda.current_stream().wait_event(loss_done)
        self.grads.finish(B["loss"])
        for l in range(L):
            _check(lib_.mcf_sgd_grow(self.W[l].data_ptr(), nc, gv[2 * l].data_ptr(), self.W[l].numel() // nc,
                                     C.c_float(self.lr), s))
            _check(lib_.mcf_sgd_grow(self.b[l].data_ptr(), nc, gv[2 * l + 1].data_ptr(), self.b[l].numel() // nc,
                                     C.c_float(self.lr), s))
        return B["loss"]

    def capture(self, xt: torch.Tensor, labels: torch.Tensor, n_global: int):
        """The step on (xt, labels) as a CUDA graph: returns replay(), which runs
        one training step on the CURRENT contents of xt / labels (refill them in
        place for a new batch) and returns the loss-terms tensor like step().
        The graph holds the step's ~50 launches over three streams, so the
        launch overhead is paid once (config 3: 1.45 -> 1.36 ms per step);
        results are the bits of step().  Single process only: the gradient
        all-reduce of a multi-rank job is left to direct step() calls.  capture()
        itself performs two real training steps (warm-up on the capture stream)."""
        if self.grads.world() > 1:
            raise RuntimeError("MCMLP.capture: multi-rank steps are not captured (NCCL all-reduce inside)")
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            # two real training steps on the capture stream first: they size
            # every buffer and the library's per-stream workspaces, so the
            # captured step allocates nothing
            self.step(xt, labels, n_global)
            self.step(xt, labels, n_global)
            stream.synchronize()
            with torch.cuda.graph(graph, stream=stream):
                loss = self.step(xt, labels, n_global)
        torch.cuda.current_stream().wait_stream(stream)

        def replay():
            graph.replay()
            return loss

        return replay

    @staticmethod
    def loss_value(loss_sum: torch.Tensor, n_global: int) -> float:
        """fl_div(sum of terms, N) in binary32 (autodiff.hpp:575) -- on the host,
        where the step's result is read anyway (a device scalar division by a
        Python number may be evaluated as a multiplication by its reciprocal)."""
        return float(np.float32(loss_sum.item()) / np.float32(n_global))

    def checkpoint(self) -> dict:
        """The model's checkpoint blob, identical to the reference's (nn.hpp:207-214)."""
        return checkpoint_to_json(self.dims, self.params_numpy(), self.nc)

    def load_checkpoint(self, ckpt: dict) -> None:
        """Restore the MC parameters bit-exact (nn.hpp:216-229)."""
        for l, (w, b) in enumerate(load_checkpoint(self.dims, ckpt, self.nc)):
            self.W[l].copy_(torch.from_numpy(w))
            self.b[l].copy_(torch.from_numpy(b))

    def params_numpy(self):
        torch.cuda.synchronize()
        return [(w.cpu().numpy(), b.cpu().numpy()) for w, b in zip(self.W, self.b)]


def model_config(dims, nc=2):
    """MCSequential.config() of the MC-MLP (nn.hpp:74-80, 135, 190-194):
    MCLinear layers with ReLU between them."""
    layers = []
    for l in range(len(dims) - 1):
        layers.append({"type": "mclinear", "in": int(dims[l]), "out": int(dims[l + 1]), "bias": True, "nc": int(nc)})
        if l + 2 < len(dims):
            layers.append({"type": "relu"})
    return {"type": "sequential", "layers": layers}


def checkpoint_to_json(dims, params, nc=2) -> dict:
    """checkpoint_to_json (nn.hpp:207-214): the topology manifest plus one mct
    blob per parameter, named as MCSequential names them ("<layer index>.weight",
    "<layer index>.bias"; ReLU layers hold no parameters).  params: list of
    (W (out, in, nc), b (out, nc)) arrays or tensors, binary32 components."""
    from . import serialize

    blobs = {}
    for l, (w, b) in enumerate(params):
        idx = 2 * l  # a ReLU follows every layer but the last
        w = torch.as_tensor(np.asarray(w.cpu() if torch.is_tensor(w) else w))
        b = torch.as_tensor(np.asarray(b.cpu() if torch.is_tensor(b) else b))
        blobs[f"{idx}.weight"] = serialize.mct_to_json(w)
        blobs[f"{idx}.bias"] = serialize.mct_to_json(b)
    return {"format": "mcf-checkpoint", "model": model_config(dims, nc), "params": blobs}


def load_checkpoint(dims, ckpt: dict, nc=2):
    """load_checkpoint (nn.hpp:216-229): the reference's checks and messages,
    then the parameters bit-exact: list of (W, b) numpy arrays."""
    from . import serialize

    if not isinstance(ckpt, dict) or ckpt.get("format", "") != "mcf-checkpoint":
        raise ValueError("load_checkpoint: not a checkpoint blob")
    if ckpt.get("model") != model_config(dims, nc):
        raise ValueError("load_checkpoint: model topology mismatch")
    out = []
    for l in range(len(dims) - 1):
        idx = 2 * l
        w = serialize.mct_from_json(ckpt["params"][f"{idx}.weight"], "b32").numpy()
        b = serialize.mct_from_json(ckpt["params"][f"{idx}.bias"], "b32").numpy()
        out.append((w, b))
    return out


__all__ = ["init_params", "make_batch", "GradExchange", "MCMLP", "SEQUENTIAL", "FAST", "model_config",
           "checkpoint_to_json", "load_checkpoint"]
