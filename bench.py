#!/usr/bin/env python
"""Benchmark of the MCF operator hot path on B200 (driver contract).

Headline workload (BASELINE.json metric "MC mm effective GFLOP/s (2MNK/t)"):
config 2 -- A = 4096 x 4096 MCTensor (nc=2, binary32 components split from
binary64 U[-1,1]) times B = 4096 x 4096 binary32 U[-1,1], plan MCF_FAST.
A "step" is one full 4096^3 MC x Tensor product; with N ranks the output rows
are sharded (strong scaling, no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (one process per GPU, NCCL).

The JSON line carries, besides the contract keys:
  roofline       the dominant kernel (the hand-written tcgen05 residue GEMM)
                 against the int8 rate implied by MEASURED_PEAKS.json, and every
                 other kernel of the step against measured HBM bandwidth
  cpu_baseline   the reference's own C++ (oracle/_ref, compiled from
                 /root/reference) on this box's host cores, bounded sample
  parity         sampled outputs of the timed product against the reference's
                 outputs and a binary128 truth (untimed)
  e2e            the same metric through the reference-facing host-buffer C-ABI
                 (mcf_h_bmm_mcn) from pinned host memory, copies included
  elementwise    config 0 operator suite (2^24 elements, fp32 nc=2)
  other_configs  configs 1a, 1b, 3, 4 (sharded across the ranks) each with its
                 own CPU baseline
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = K = N = 4096
METRIC = "MC mm effective GFLOP/s (2MNK/t)"
UNIT = "GFLOP/s"
WORKLOAD = "config2: MC(4096x4096, nc=2, fp32) x T(4096x4096, fp32)"
L2_NOTE = "256 MiB buffer written between timed steps"


def grid_for(world):
    """Output-block grid (row blocks, column blocks) of the ranks; MCF_BENCH_GRID=rows keeps plain row shards."""
    from paper_2207_08867_b200.dist import block_grid

    return (world, 1) if os.environ.get("MCF_BENCH_GRID") == "rows" else block_grid(world)


def config_dict(world):
    """The workload description, identical in both arms."""
    gr, gc = grid_for(world)
    par = "1 GPU" if world == 1 else (f"output rows / {world} GPUs" if gc == 1 else
                                      f"output blocks, {gr} row blocks x {gc} column blocks / {world} GPUs")
    return {"workload": WORKLOAD, "M": M, "K": K, "N": N, "nc": 2, "parallelism": par, "l2": L2_NOTE}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ncu_traffic():
    """DRAM bytes per launch of the GEMM from the committed ncu --set full
    capture (profiles/ncu_traffic_r*.json, newest round), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_r*.json")))
    if not files:
        return None, None
    d = json.load(open(files[-1]))
    return d.get("traffic_bytes_per_launch"), os.path.relpath(files[-1], ROOT)


# ---- clocks during the timed region -------------------------------------------------

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.summary = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if not self.proc:
            return
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if sm:
            busy = [s for s in sm if s > 0.5 * max(sm)] or sm
            self.summary = {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                            "samples": len(sm)}


# ---- the reference side (oracle/_ref only: never loads the product library) ---------

def ref_split(v, nc, dtype):
    """expansion_of_double (mc_ops.hpp:286-297): greedy round-and-residual."""
    import numpy as np

    rest = np.asarray(v, np.float64).copy()
    out = np.zeros(rest.shape + (nc,), dtype)
    for i in range(nc):
        c = rest.astype(dtype)
        out[..., i] = c
        rest = rest - c.astype(np.float64)
    return out


def ref_config2(ref, rows=M):
    """Config 2's inputs from the reference's own Rng (rng.hpp) -- identical to
    paper_2207_08867_b200.data.config2 (pinned by tests/test_rng_pin.py).
    Only the first `rows` rows of A are materialised."""
    import numpy as np

    a = ref_split(-1.0 + 2.0 * ref.rng_uniform(2000, rows * K), 2, np.float32).reshape(rows, K, 2)
    b = (-1.0 + 2.0 * ref.rng_uniform(2001, K * N)).astype(np.float32).reshape(K, N)
    return a, b


def reference_sample(a, b, threads):
    """The reference's mm_mcn (oracle/_ref) on `threads` full output rows of the
    config-2 product, one row per thread: (GFLOP/s, seconds, rows, kind, out)."""
    import oracle

    rows = max(threads, 1)
    if oracle.ref_available():
        t, out = oracle.Oracle("ref").time_mm_rows(a[:rows], b, rows, threads=threads)
        kind = "reference"
    else:  # the reference tree did not compile here: the C port, one thread per row
        import concurrent.futures as cf

        port = oracle.Oracle("port")
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(lambda r: port.mm_mcn(a[r:r + 1], b), range(rows)))
        t = time.perf_counter() - t0
        import numpy as np

        out = np.concatenate(parts, 0)
        kind = "port"
    return 2.0 * rows * K * N / t / 1e9, t, rows, kind, out


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle

    threads = cpu_threads()
    if oracle.ref_available():
        a, b = ref_config2(oracle.Oracle("ref"), rows=threads)
    else:
        # the reference tree did not compile here: the oracle's C port is timed
        # instead (reference_sample, kind "port"), on inputs from the pinned
        # restatement of the reference's Rng mappings (tests/test_rng_pin.py)
        from paper_2207_08867_b200 import data

        a_full, b = data.config2(M, K, N)
        a = a_full[:threads]
    for _ in range(args.warmup):
        reference_sample(a, b, threads)
    vals, secs = [], []
    kind = "reference"
    for _ in range(args.steps):
        v, t, rows, kind, _ = reference_sample(a, b, threads)
        vals.append(v)
        secs.append(t)
    value = statistics.mean(vals)
    sample = f"{threads} full output rows (x {K} x {N}) of the 4096^3 product per step, one row per host thread"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(secs), 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (the reference's emulation of binary32 components)", "data": "synthetic",
        "config": config_dict(world),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baselines_other(a2, b2):
    """The reference's own C++ on this box's cores for configs 0, 1a, 1b, 3, 4
    (bounded samples, a few seconds each; units as each config reports)."""
    import numpy as np

    import oracle

    if not oracle.ref_available():
        return None
    ref = oracle.Oracle("ref")
    thr = cpu_threads()
    res = {}
    # config 0: 2^22 elements per operator (all cores, disjoint slices)
    n0 = 1 << 22
    u = lambda seed, n: (-1.0 + 2.0 * ref.rng_uniform(seed, 2 * n)[0::2]) * np.exp2(-8.0 + 16.0 * ref.rng_uniform(seed, 2 * n)[1::2])
    xv, yv = u(1000, n0), u(1001, n0)
    x, y = ref_split(xv, 2, np.float32), ref_split(yv, 2, np.float32)
    yd = ref_split(yv + np.sign(yv) * 0.5, 2, np.float32)
    v = u(1002, n0).astype(np.float32)
    xe = ref_split(np.clip(u(1003, n0), -10.0, 10.0), 2, np.float32)
    ops = {"grow_expn": (dict(x=x, v=v), 20), "scaling_n": (dict(x=x, v=v), 20), "div_n": (dict(y=yd, v=v), 20),
           "add_mcn": (dict(x=x, y=y), 24), "mul_mcn": (dict(x=x, y=yd), 24), "div_mcn": (dict(x=x, y=yd), 24),
           "exp_mcn": (dict(x=xe), 16), "square_mcn": (dict(x=x), 16), "mul_mcn_slow": (dict(x=x, y=y), 24)}
    c0 = {}
    for op, (kw, bpe) in ops.items():
        t, _ = ref.time_elementwise(op, threads=thr, **kw)
        c0[op] = {"GB/s": round(bpe * n0 / t / 1e9, 3), "ns_per_elem_per_core": round(t * thr / n0 * 1e9, 1)}
    res["config0"] = {"sample": f"2^22 elements per operator, {thr} threads", "cores": thr, "kind": "reference", "ops": c0}
    # config 1a: matvec rows (MC nc=3 x T vector): 4096 rows of 4096
    rows = 4096
    x3 = ref_split(u(1100, rows * K), 3, np.float32).reshape(rows, K, 3)
    vec = u(1101, K).astype(np.float32).reshape(K, 1)
    t, _ = ref.time_mm_rows(x3, vec, rows, threads=thr)
    res["config1a_mv_nc3"] = {"GMAD/s": round(rows * K / t / 1e9, 4), "cores": thr, "kind": "reference",
                              "sample": f"{rows} of 65536 rows (x 4096 MADs)"}
    # config 1b: 4096 of the 65536 MC x MC dots (recipe B)
    y3 = ref_split(u(1102, rows * K), 3, np.float32).reshape(rows, K, 3)
    t, _ = ref.time_dot_mcmc(x3, y3, threads=thr)
    res["config1b_dots_mcmc_nc3"] = {"GMAD/s": round(rows * K / t / 1e9, 4), "cores": thr, "kind": "reference",
                                     "sample": f"{rows} of 65536 dots (x 4096 MADs), recipe B"}
    # config 4: 256 sampled outputs (dots of K = 16384) per variant
    k4, s4 = 16384, 256
    for tag, dt, nc, sc in (("fp32_nc2", np.float32, 2, 1.0), ("fp16_nc3", np.float16, 3, 1.0 / 64)):
        xa = ref_split((-1.0 + 2.0 * ref.rng_uniform(4000, s4 * k4)) * sc, nc, dt).reshape(s4, k4, nc)
        ya = ref_split((-1.0 + 2.0 * ref.rng_uniform(4001, s4 * k4)) * sc, nc, dt).reshape(s4, k4, nc)
        t, _ = ref.time_dot_mcmc(xa, ya, threads=thr)
        res[f"config4_mcmc_{tag}"] = {"GFLOP/s_eff": round(2.0 * s4 * k4 / t / 1e9, 4), "cores": thr,
                                      "kind": "reference", "sample": f"{s4} outputs of the 16384^3 product (recipe B)"}
    # config 3: the reference's own training loop, one step at a reduced batch
    dims = [784, 1024, 1024, 10]
    nb = 8
    counts = [dims[l + 1] * dims[l] + dims[l + 1] for l in range(3)]
    uu = ref.rng_uniform(3000, sum(counts))
    params, off = [], 0
    for l in range(3):
        fan, outd = dims[l], dims[l + 1]
        bd = 1.0 / np.sqrt(float(fan))
        w = -bd + 2.0 * bd * uu[off:off + outd * fan]
        off += outd * fan
        bb = -bd + 2.0 * bd * uu[off:off + outd]
        off += outd
        params.append((ref_split(w, 2, np.float32).reshape(outd, fan, 2), ref_split(bb, 2, np.float32).reshape(outd, 2)))
    X = ref.rng_normal(3001, nb * 784).astype(np.float32).reshape(nb, 784)
    lab = ref.rng_below(3002, 10, nb).astype(np.int32)
    t0 = time.perf_counter()
    oracle.mlp_train_reference(dims, 2, params, X, lab, 1, 0.01)
    t = time.perf_counter() - t0
    res["config3_mlp"] = {"ms_per_step_at_batch_8192": round(t * 8192 / nb * 1e3, 1), "cores": 1, "kind": "reference",
                          "sample": f"one training step at batch {nb} (the reference's loop is single-threaded), "
                                    "scaled to 8192"}
    return res


# ---- our arm ---------------------------------------------------------------------

def _dev_time(torch, fn, reps, flush=None, world=1):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    from paper_2207_08867_b200.dist import max_over_ranks

    return max_over_ranks(statistics.median(ts), device="cuda")


def elementwise_suite(torch, mcf, hbm_gbs, rank=0, world=1):
    """Config 0 (2^24 elements, fp32 nc=2): device time per operator.  With
    world > 1 every rank takes its flat range (no collective); the time is the
    max over ranks and the GB/s the whole job's.  `us` is one launch after an
    L2 flush; `us_b2b` the mean of 20 back-to-back launches (every launch's
    dirty output lines are written back within the run)."""
    from paper_2207_08867_b200 import data
    from paper_2207_08867_b200.dist import max_over_ranks, row_range

    n = 1 << 24
    lo, hi = row_range(n, rank, world)
    x, y, yd, v, xe = (torch.from_numpy(t[lo:hi]).cuda() for t in data.config0(n))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ops = {
        "grow_expn": (lambda: mcf.grow_expn(x, v), 20), "scaling_n": (lambda: mcf.scaling_n(x, v), 20),
        "div_n": (lambda: mcf.div_n(v, yd), 20), "add_mcn": (lambda: mcf.add_mcn(x, y), 24),
        "mul_mcn": (lambda: mcf.mul_mcn(x, yd), 24), "div_mcn": (lambda: mcf.div_mcn(x, yd), 24),
        "exp_mcn": (lambda: mcf.exp_mcn(xe), 16), "square_mcn": (lambda: mcf.square_mcn(x), 16),
        "mul_mcn_slow": (lambda: mcf.mul_mcn_slow(x, y), 24),
    }
    res = {}
    for name, (f, bpe) in ops.items():
        ms = _dev_time(torch, f, 5, flush, world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        b2b = max_over_ranks(e0.elapsed_time(e1) / 20, device="cuda")
        gbs = bpe * n / ms / 1e6
        res[name] = {"us": round(ms * 1e3, 1), "GB/s": round(gbs, 1), "frac_hbm": round(gbs / hbm_gbs / world, 3),
                     "us_b2b": round(b2b * 1e3, 1), "frac_hbm_b2b": round(bpe * n / b2b / 1e6 / hbm_gbs / world, 3),
                     "bytes_per_elem": bpe}
    del x, y, yd, v, xe, flush
    return res


def other_configs(torch, mcf, hbm_gbs, rank, world):
    """BASELINE configs 1, 3 and 4, sharded as SURVEY 8e says: 1a by rows, 1b
    by dot index, 3 data-parallel (NCCL all-reduce of the binary32 gradients),
    4 by output rows with B broadcast once from rank 0 (untimed).  Inputs are
    drawn on the device (torch CUDA generator, seeded) with each config's
    distribution; parity for these paths is in tests/.  Times: max over ranks."""
    import numpy as np

    from paper_2207_08867_b200 import mlp
    from paper_2207_08867_b200.dist import broadcast_, row_range

    g = torch.Generator(device="cuda").manual_seed(2207 + rank)
    res = {}

    def cfg0_dist(shape, nc, dtype=torch.float32, scale=1.0):
        v = (torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1)
        v = v * torch.exp2(torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) * 16 - 8) * scale
        comps = []
        for _ in range(nc):
            c = v.to(dtype)
            comps.append(c)
            v = v - c.to(torch.float64)
        return torch.stack(comps, -1).contiguous()

    # config 1a: MC (65536 x 4096, nc=3) x T vector, FAST (HBM-bound); rows sharded
    M1, K1 = 65536, 4096
    r0, r1 = row_range(M1, rank, world)
    x = cfg0_dist((r1 - r0, K1), 3)
    v = cfg0_dist((K1,), 1)[..., 0].contiguous()
    broadcast_(v)
    ms = _dev_time(torch, lambda: mcf.mv_mcn(x, v, plan=mcf.FAST), 5, world=world)
    byts = M1 * K1 * 12 + K1 * 4 + M1 * 12
    res["config1a_mv_nc3"] = {"shape": [M1, K1, 3], "ms": round(ms, 4), "GB/s": round(byts / ms / 1e6, 1),
                              "frac_hbm": round(byts / ms / 1e6 / hbm_gbs / world, 3),
                              "GMAD/s": round(M1 * K1 / ms / 1e6, 1), "sharding": f"rows / {world}"}
    # config 1b: 65536 independent MC x MC dots (length 4096, nc=3); dot index sharded
    y = cfg0_dist((r1 - r0, K1), 3)
    ms = _dev_time(torch, lambda: mcf.dot_mcmc(x, y, plan=mcf.FAST), 5, world=world)
    byts = 2 * M1 * K1 * 12 + M1 * 12
    res["config1b_dots_mcmc_nc3"] = {"shape": [M1, K1, 3], "ms": round(ms, 4), "GB/s": round(byts / ms / 1e6, 1),
                                     "frac_hbm": round(byts / ms / 1e6 / hbm_gbs / world, 3),
                                     "sharding": f"dots / {world}"}
    del x, y, v
    torch.cuda.empty_cache()
    # config 3: MC-MLP 784-1024-1024-10, nc=2, global batch 8192, MC-SGD lr 0.01;
    # data parallel: each rank 8192 / world samples, gradients summed by NCCL
    dims, nglob = [784, 1024, 1024, 10], 8192
    params = mlp.init_params(dims, 2)
    xb, yb = mlp.make_batch(nglob)
    s0, s1 = row_range(nglob, rank, world)
    group = torch.distributed.group.WORLD if world > 1 else None
    model = mlp.MCMLP(dims, params, lr=0.01, plan=mcf.FAST, group=group)
    xt = torch.from_numpy(np.ascontiguousarray(xb[s0:s1].T)).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(yb[s0:s1])).cuda()
    first = model.loss_value(model.step(xt, yt, nglob), nglob)
    # one process: the step replayed as a CUDA graph (~50 launches over three
    # streams; same bits as direct calls); several ranks: direct calls
    run_step = model.capture(xt, yt, nglob) if world == 1 else (lambda: model.step(xt, yt, nglob))
    ms = _dev_time(torch, run_step, 10, world=world)
    last = model.loss_value(run_step(), nglob)
    res["config3_mlp"] = {"dims": dims, "batch": nglob, "ms_per_step": round(ms, 3),
                          "steps_per_s": round(1e3 / ms, 2), "loss_first": first,
                          f"loss_after_{16 if world == 1 else 14}_steps": last,
                          "launch": "CUDA graph replay of the step" if world == 1 else "direct calls",
                          "sharding": f"data parallel / {world}, NCCL all-reduce of 1,863,690 binary32 gradients"}
    del model, xt, yt
    torch.cuda.empty_cache()
    # config 4: MC x MC 16384^3, fp32 nc=2 and fp16 nc=3 (values U[-1,1]/64);
    # output rows sharded, B replicated by a one-time broadcast from rank 0
    N4 = 16384
    q0, q1 = row_range(N4, rank, world)
    for tag, dtype, nc, scale, reps in (("fp32_nc2", torch.float32, 2, 1.0, 2), ("fp16_nc3", torch.float16, 3, 1 / 64, 3)):
        def split(v):
            comps = []
            for _ in range(nc):
                c = v.to(dtype)
                comps.append(c)
                v = v - c.to(torch.float64)
            return torch.stack(comps, -1).contiguous()

        a = split((torch.rand((q1 - q0, N4), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * scale)
        b = split((torch.rand((N4, N4), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * scale)
        broadcast_(b)  # one-time, untimed
        ms = _dev_time(torch, lambda: mcf.mm_mcmc(a, b, plan=mcf.FAST), reps, world=world)
        gemms = mcf.lib().mcf_fast_tc_gemm_equivalents(2, N4) if nc == 2 else 15
        entry = {"M=N=K": N4, "ms": round(ms, 2), "GFLOP/s_eff": round(2 * N4 ** 3 / ms / 1e6, 1),
                 "int8_gemms": gemms, "int8_TOPS_step": round(2 * N4 ** 3 * gemms / (ms * 1e-3) / 1e12, 1),
                 "sharding": f"rows / {world}, B broadcast once"}
        entry["path"] = ("int8 tensor cores, CRT over %d moduli (tcgen05)" % gemms if nc == 2 else
                         "int8 tensor cores, five digits per pre-summed element (15 GEMM-equivalents)")
        res[f"config4_mcmc_{tag}"] = entry
        del a, b
        torch.cuda.empty_cache()
    return res


def run_ours(args, N_ALL=N):
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2207_08867_b200 as mcf
    from paper_2207_08867_b200 import data
    from paper_2207_08867_b200.dist import block_range, max_over_ranks

    rank, world, local = env_rank()
    # MCF_BENCH_SHARE_GPU=1 MCF_BENCH_BACKEND=gloo: a plumbing rehearsal of the
    # multi-rank flow on ONE GPU (all ranks on cuda:0, gloo collectives) --
    # exercises the sharding, barriers and gathers, never used for numbers
    if os.environ.get("MCF_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("MCF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6446.6))

    # inputs: generated on the host from the reference's Rng mappings, resident in HBM
    # the rank's output block: its rows of A and its columns of B (N below is
    # the block's width; the whole-job flops use M_ALL x N_ALL)
    a_h, b_full = data.config2(M, K, N_ALL)
    r0, r1, c0, c1 = block_range(M, N_ALL, rank, world, grid_for(world))
    rows = r1 - r0
    N = c1 - c0  # noqa: N806 -- the block's width shadows the module constant inside this function
    b_h = np.ascontiguousarray(b_full[:, c0:c1])
    a = torch.from_numpy(a_h[r0:r1]).cuda()
    b = torch.from_numpy(b_h).cuda()
    out = torch.empty((rows, N, 2), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    stream = torch.cuda.current_stream()

    def step():
        rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, rows, K, N, 0, out.data_ptr(),
                             mcf.FAST, 1, stream.cuda_stream)
        if rc != 0:
            raise RuntimeError(lib.mcf_last_error().decode())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mcf.reset_launch_count()
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for e0, e1 in ev:
            flush.zero_()  # L2 flush between steps (outside the event pair)
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = mcf.launch_count()
    times = [e0.elapsed_time(e1) for e0, e1 in ev]
    ms = max_over_ranks(sum(times) / len(times), device="cuda")
    value = 2.0 * M * N_ALL * K / (ms * 1e-3) / 1e9

    # ---- roofline: the dominant kernel is the residue GEMM (one launch per
    # product, batched over the moduli).  Algorithmic int8 ops per launch:
    # 2 rows N Kp x moduli; its device time from CUDA events around the GEMM
    # phase on the launching stream (mcf_fast_mm_phases), median of 5.
    n_mod = lib.mcf_fast_tc_gemm_equivalents(1, K)
    kp = (K + 31) // 32 * 32
    int8_ops = 2.0 * rows * N * kp * n_mod
    phases = []
    fb = C.c_int64(0)
    for _ in range(5):
        ph = (C.c_double * 4)()
        flush.zero_()
        rc = lib.mcf_fast_mm_phases(a.data_ptr(), b.data_ptr(), rows, K, N, out.data_ptr(), ph, C.byref(fb),
                                    stream.cuda_stream)
        if rc != 0:
            raise RuntimeError(lib.mcf_last_error().decode())
        phases.append(list(ph))
    med = [statistics.median(p[i] for p in phases) for i in range(4)]
    gemm_ms = med[2]
    achieved = int8_ops / (gemm_ms * 1e-3) / 1e12
    # int8 denominator: MEASURED_PEAKS.json holds the measured dense bf16 rate;
    # B200's dense int8 rate is twice its dense bf16 rate, so 2 x the measured
    # burst figure (the GEMM is timed as one ~0.7 ms launch: burst, not sustained)
    peak_i8 = 2.0 * float(pk.get("bf16_tflops", 1627.0))
    # the other kernels of the step against measured HBM (algorithmic bytes)
    mpad, npad = rows, (N + 15) // 16 * 16
    b_bytes = K * N * 4 + n_mod * npad * kp + K * N * 4   # read B, residue planes, transposed copy
    a_bytes = rows * K * 8 * 2 + n_mod * rows * kp         # row maxima pass + residue pass read A, planes
    c_bytes = n_mod * rows * npad + rows * N * 8           # residue planes in, two components out
    kernels = {
        "b_residues": {"ms": round(med[0], 4), "bytes": b_bytes, "frac_hbm": round(b_bytes / med[0] / 1e6 / hbm, 3)},
        "a_residues": {"ms": round(med[1], 4), "bytes": a_bytes, "frac_hbm": round(a_bytes / med[1] / 1e6 / hbm, 3),
                       "note": "side stream, overlapped with b_residues in the timed step"},
        "residue_gemm": {"ms": round(gemm_ms, 4), "TOPS": round(achieved, 1), "frac_int8": round(achieved / peak_i8, 3)},
        "crt_reconstruction_and_fallback": {"ms": round(med[3], 4), "bytes": c_bytes,
                                            "frac_hbm": round(c_bytes / med[3] / 1e6 / hbm, 3),
                                            "fallback_outputs": int(fb.value)},
    }

    # context: the same product on the FP64 pipe (MCF_FAST_FP64, offset accumulation)
    def step64():
        rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, rows, K, N, 0, out.data_ptr(),
                             mcf.FAST_FP64, 1, stream.cuda_stream)
        if rc != 0:
            raise RuntimeError(lib.mcf_last_error().decode())

    step64()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(2):
        step64()
    e1.record(stream)
    torch.cuda.synchronize()
    ms64 = max_over_ranks(e0.elapsed_time(e1) / 2, device="cuda")
    f64 = C.c_double(0.0)
    f32 = C.c_double(0.0)
    lib.mcf_probe_pipe_rates(C.byref(f64), C.byref(f32))
    ops64 = lib.mcf_fast_ops_per_mad(0, mcf.B32, 2)
    fp64_path = {"ms_per_step": round(ms64, 3), "GFLOP/s_eff": round(2.0 * M * N_ALL * K / ms64 / 1e6, 1),
                 "fp64_ops_per_mad": ops64, "fp64_pipe_TFLOPs": round(ops64 * rows * N * K / ms64 / 1e9, 3),
                 "fp64_pipe_peak_measured": round(f64.value / 1e12, 3)}
    step()  # leave `out` holding the headline path's result (for the parity stamp)
    torch.cuda.synchronize()
    out_h = out.cpu().numpy() if rank == 0 else None

    # ---- e2e through the host-buffer C-ABI, pinned buffers, copies inside the timed region
    a_pin = torch.from_numpy(a_h[r0:r1]).pin_memory()
    b_pin = torch.from_numpy(b_h).pin_memory()
    o_pin = torch.empty((rows, N, 2), dtype=torch.float32).pin_memory()
    e2e_steps = max(3, args.steps // 2)

    def e2e_step():
        rc = lib.mcf_h_bmm_mcn(mcf.B32, a_pin.data_ptr(), 2, b_pin.data_ptr(), 1, rows, K, N, 0,
                               o_pin.data_ptr(), mcf.FAST)
        if rc != 0:
            raise RuntimeError(lib.mcf_last_error().decode())

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, device="cuda")
    e2e_val = 2.0 * M * N_ALL * K / e2e_s / 1e9
    h2d_bytes = int(a_pin.numel() * 4 + b_pin.numel() * 4)
    d2h_bytes = int(o_pin.numel() * 4)

    del a, b, out, a_pin, b_pin, o_pin, flush
    torch.cuda.empty_cache()
    ew = elementwise_suite(torch, mcf, hbm, rank, world)  # flat-range shards across ranks
    others = None if args.no_extras else other_configs(torch, mcf, hbm, rank, world)

    cpu = parity = cpu_other = None
    if rank == 0 and world == 1:
        # CPU baseline (the reference compiled here) on this box's cores; the
        # rows it computes double as the parity sample of the timed product
        gf, t, nrows, kind, ref_out = reference_sample(a_h, b_h, cpu_threads())
        cpu = {"value": round(gf, 4), "unit": UNIT, "cores": cpu_threads(), "kind": kind,
               "sample": f"{nrows} full output rows of the 4096^3 product, one row per host thread ({t:.1f} s)"}
        import oracle

        port = oracle.Oracle("port")
        rng = np.random.default_rng(7)
        ri, ci = rng.integers(0, nrows, 2048), rng.integers(0, N, 2048)
        ge = port.relerr_mm_mct(a_h, b_h, ri, ci, out_h[ri, ci])
        re_ = port.relerr_mm_mct(a_h, b_h, ri, ci, ref_out[ri, ci])
        lg = lambda v: round(float(np.log2(max(v, 1e-300))), 2)
        parity = {"sample": f"2048 outputs of the timed product (rows 0..{nrows - 1}) vs binary128 truth",
                  "gpu_median_log2": lg(np.median(ge)), "gpu_max_log2": lg(ge.max()),
                  "reference_median_log2": lg(np.median(re_)), "reference_max_log2": lg(re_.max()),
                  "within_4x_of_reference": bool(np.median(ge) <= 4 * np.median(re_) and ge.max() <= 4 * re_.max())}
        if not args.no_extras:
            cpu_other = cpu_baselines_other(a_h, b_h)

    traffic, traffic_src = ncu_traffic()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "s8 residues -> s32 (exact), binary32 CRT slice sums + binary64 join; fp32 nc=2 in/out",
            "data": "synthetic (the reference's Rng mappings, seeds per SURVEY 8d)",
            "config": config_dict(world),
            "plan": "MCF_FAST",
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak_i8, 1),
                         "unit": "TOPS (int8)", "frac": round(achieved / peak_i8, 3),
                         "traffic": traffic, "traffic_unit": "bytes/launch (DRAM read+write, ncu --set full)",
                         "traffic_source": traffic_src,
                         "kernel": f"k_tc_gemm_s8 (hand-written tcgen05 kind::i8, TMA, TMEM), one launch per product "
                                   f"batched over {n_mod} moduli, int8 residue epilogue",
                         "algorithmic_int8_ops_per_launch": int8_ops,
                         "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (burst; dense int8 = 2 x dense bf16 on B200)",
                         "peak_nominal_int8": 4500.0,
                         "kernels": kernels},
            "fp64_pipe_path": fp64_path,
            "e2e": {"value": round(e2e_val, 1), "unit": UNIT,
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes},
            "gpu_launches": launches,
            "clocks": clk.summary,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if parity:
            line["parity"] = parity
        line["elementwise"] = {"config": "config0: 2^24 elements, fp32 nc=2, bit-exact vs reference"
                                         + (f", flat range over {world} GPUs" if world > 1 else ""),
                               "hbm_peak_gbs": hbm, "frac_hbm_per_gpu": True, "ops": ew}
        if others:
            if cpu_other:
                others["cpu_baselines"] = cpu_other
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip configs 1, 3, 4 (headline + config 0 only)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
