#!/usr/bin/env python
"""Benchmark of the B200 RSR / RSR++ matvec (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config NAME] [--variant rsrpp|rsr|both] [--replays R]

One JSON line on stdout (rank 0).  A "step" is one matvec v . A over the whole synthetic
matrix (one pass of the hot path over one batch: B=64 vectors for the batch config) with the
index and v already resident in HBM (`value`).  The timed region is K steps captured in one
CUDA graph; it is measured R times (default 11) and the median replay is reported
(`ms_per_step` = median / K; every replay in `timing.replays_ms`).  `e2e` is the same metric
through the reference-facing API with host buffers, in the reference's calling convention:
`rsr.multiply_ternary(numpy float64 v, idx)` (core.py:110-117 casts every vector to fp64);
the int32 host call is reported beside it (`e2e_int32`).

L2 rule: each timed step multiplies against a different copy of the index (rotating >= 4 x
L2 worth of index bytes), so no step reads an index the previous step left in L2.

Configs (BASELINE.json): ternary16384 (default, the headline), ternary4096f32 (config 1),
binary16384 (config 2: RSR and RSR++ side by side), ternary16384b64 (config 3),
llama4096 / llama4096x14336 / llama14336x4096 (config 4), ternary65536 and ternary65536s
(config 5).  Every line carries the CPU baseline (C port of the reference's RSR++ on all host
cores and on one, and its standard dense multiply on one core) unless --no-cpu.

N > 1 (torchrun): the default is weak scaling of the column-sharded matvec — rank g owns a
full n x m shard (columns [g*m, (g+1)*m) of an n x (N*m) matrix; rank 0's shard is the N=1
matrix), multiplies it, and the output slices are NCCL all-gathered every step on a comm
stream that overlaps the next step's multiply (double-buffered slices).  value = n x m
shard-matvecs per second summed over ranks (each step is one matvec of the n x N*m matrix).
`multi_gpu` reports the compute-only and compute + all-gather times separately and the check
of the gathered vector against every rank's oracle slice.  --config ternary65536s (BASELINE
config 5, strong scaling): ONE 65536 x 65536 matrix (hash-generated per entry, so every N
shards the same matrix), rank g owning column blocks [g*NB//N, (g+1)*NB//N) (the
multiply_parallel partition, kernels.py:222); value = full matvecs per second.

--impl reference: the reference algorithm's CPU path (oracle/rsr_oracle.c, a C port of
`_run_blocks` + `multiply_parallel`; the reference itself is Python + Numba and cannot travel
to the GPU box) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (domain, n rows, m cols, workload description)
    "ternary16384": ("ternary", 16384, 16384, "ternary 16384x16384 RSR++ matvec, int32-exact integer activations"),
    "binary16384": ("binary", 16384, 16384, "binary 16384x16384 matvec, RSR and RSR++ kernels"),
    "llama4096": ("ternary", 4096, 4096, "ternary 4096x4096 (Llama-3-8B q/o) RSR++ decode matvec"),
    "llama4096x14336": ("ternary", 4096, 14336, "ternary 4096x14336 (Llama-3-8B gate/up) RSR++ decode matvec"),
    "llama14336x4096": ("ternary", 14336, 4096, "ternary 14336x4096 (Llama-3-8B down) RSR++ decode matvec"),
    "ternary65536": ("ternary", 65536, 65536, "ternary 65536x65536 RSR++ matvec"),
    "ternary16384b64": ("ternary", 16384, 16384, "ternary 16384x16384 RSR++, batch of 64 int32 activation vectors"),
    "ternary4096f32": ("ternary", 4096, 4096, "ternary 4096x4096 RSR++ matvec, single fp32 vector"),
    "ternary65536s": ("ternary", 65536, 65536, "ternary 65536x65536 RSR++ matvec, column blocks sharded "
                      "across the ranks (kernels.py:222 partition) + NCCL all-gather of the output"),
}
STRONG = {"ternary65536s"}  # BASELINE config 5: one matrix split over the ranks (strong scaling)
FP32 = {"ternary4096f32"}
FP32_TOL = 1e-5  # north star: fp32 activations within 1e-5 relative (norm-wise) of the fp64 reference
BATCH = {"ternary16384b64": 64}
BOTH_VARIANTS = {"binary16384"}  # BASELINE config 2: "RSR vs RSR++ kernels"
PEAK_ADDS = 148 * 128 * 1.965e9  # int32 add lanes per second (SURVEY.md 8(d) adds/s view)
L2_BYTES = 126 * 1024 * 1024


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _profile(config: str, variant: str = "rsrpp"):
    """ncu numbers of this config's dominant kernel from the committed captures
    (profiles/ncu_summary.json, written by tools/summarize_ncu.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        if config == "ternary65536s" and int(os.environ.get("WORLD_SIZE", "1")) == 1:
            config = "ternary65536"  # at N = 1 the strong shard is the whole 65536^2 matrix: the same launch
        return s.get(config if variant == "rsrpp" else f"{config}:{variant}", {})
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def clocks_bad(cs) -> bool:
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(cs["reasons"])
    stuck = bool(cs["sm_mhz"] and cs["sm_max_mhz"] and cs["sm_mhz"] < 0.8 * cs["sm_max_mhz"] and not cs["reasons"])
    return bool(bad) or stuck


def make_matrix(domain: str, n: int, m: int, seed: int = 0) -> np.ndarray:
    """Reference convention (bench.py:80-84): default_rng([seed, n, m]) uniform entries."""
    rng = np.random.default_rng([seed, n, m])
    if domain == "ternary":
        return rng.integers(-1, 2, size=(n, m), dtype=np.int8)
    return rng.integers(0, 2, size=(n, m), dtype=np.int8)


def hashed_ternary(n: int, c0: int, c1: int, m_total: int, seed: int = 0):
    """Columns [c0, c1) of an n x m_total uniform ternary matrix whose entry (i, j) is a hash of
    (seed, i * m_total + j): every shard split of the same matrix gets the same entries
    (strong-scaling config).  Built on the GPU in row chunks; returns a CUDA int8 tensor."""
    import torch
    M = torch.empty((n, c1 - c0), dtype=torch.int8, device="cuda")
    cols = torch.arange(c0, c1, dtype=torch.int64, device="cuda")
    mask = (1 << 62) - 1
    for r0 in range(0, n, 4096):
        r1 = min(n, r0 + 4096)
        x = torch.arange(r0, r1, dtype=torch.int64, device="cuda")[:, None] * m_total + cols[None, :]
        x = (x + seed * 0x5851F42D4C957F2D + 0x14057B7EF767814F) & mask
        for mul in (0x2545F4914F6CDD1D, 0x1B873593):  # xorshift-multiply rounds (63-bit lanes)
            x = ((x ^ (x >> 29)) * mul) & mask
        M[r0:r1] = (((x >> 20) % 3) - 1).to(torch.int8)
    return M


def make_vector(n: int, seed: int = 0) -> np.ndarray:
    """Integer activations in [-100, 100] (bench.py:85)."""
    return np.random.default_rng([seed, n, 1]).integers(-100, 101, size=n).astype(np.int32)


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _time_calls(run, budget_s: float, min_reps: int = 3):
    """bench.py:35-43 semantics: 3 warm-ups, then perf_counter samples until the budget."""
    for _ in range(3):
        run()
    samples = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(samples) < min_reps:
        t0 = time.perf_counter()
        run()
        samples.append(time.perf_counter() - t0)
    return float(np.mean(samples)), len(samples)


def cpu_baseline(A: np.ndarray, v: np.ndarray, k: int, domain: str, variant: str, budget_s: float, batch: int = 1):
    """SURVEY.md §8(d) CPU baseline, on this box's host cores: the C port of the reference's
    `multiply_parallel` (kernels.py:209-239) with W = all host threads (the line's `value`) and
    W = 1, and the standard dense multiply (core.py:135-169, C port `naive_ternary`) on one
    core.  fp64, the reference's type.  B = 64 = 64 sequential single-vector calls (the
    reference has no batch API): timed per call."""
    from oracle import c_oracle
    n, m = A.shape
    kp = c_oracle.keys_ternary(A, k, 1)
    kn = c_oracle.keys_ternary(A, k, -1) if domain == "ternary" else None
    v64 = v.astype(np.float64)
    fold = variant != "rsr"
    W = cpu_threads()
    t_all, r_all = _time_calls(lambda: c_oracle.multiply_parallel(v64, kp, kn, m, k, fold, W), budget_s * 0.5)
    t_one, r_one = _time_calls(lambda: c_oracle.multiply_parallel(v64, kp, kn, m, k, fold, 1), budget_s * 0.25, 1)
    t_std, r_std = _time_calls(lambda: c_oracle.naive_ternary(v64, A), budget_s * 0.25, 1)
    name = "RSR++" if fold else "RSR"
    return {"value": 1.0 / t_all, "unit": "vectors/s", "cores": W, "kind": "port",
            "sample": f"{r_all} full {n}x{m} {name} matvecs (k={k}, fp64, C port of kernels.py:127-239 "
                      f"multiply_parallel on {W} threads)" + (f"; batch {batch} = {batch} sequential calls" if batch > 1 else ""),
            f"{variant}_1thread": {"value": 1.0 / t_one, "unit": "vectors/s", "cores": 1, "reps": r_one},
            "standard_1thread": {"value": 1.0 / t_std, "unit": "vectors/s", "cores": 1, "reps": r_std,
                                 "what": "naive_multiply (core.py:135-169), C port"}}


def run_reference(args, cfg):
    """--impl reference: rank 0 only, the C port of the reference CPU path."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    domain, n, m, desc = cfg
    from paper_2411_06360_b200.indexer import optimal_k_rsrpp
    k = args.k or optimal_k_rsrpp(n)
    A = make_matrix(domain, n, m)
    v = (np.random.default_rng([0, n, 2]).standard_normal(n).astype(np.float32) if args.config in FP32
         else make_vector(n))
    from oracle import c_oracle
    workers = cpu_threads()
    kp = c_oracle.keys_ternary(A, k, 1)
    kn = c_oracle.keys_ternary(A, k, -1) if domain == "ternary" else None
    v64 = v.astype(np.float64)
    fold = _variants(args)[0] != "rsr"
    for _ in range(max(args.warmup, 0)):
        c_oracle.multiply_parallel(v64, kp, kn, m, k, fold, workers)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        c_oracle.multiply_parallel(v64, kp, kn, m, k, fold, workers)
    dt = (time.perf_counter() - t0) / args.steps
    value = 1.0 / dt
    line = {
        "impl": "reference", "metric": _metric(domain), "value": value,
        "unit": "vectors/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": _config_key(args, cfg, k),
        "cpu_baseline": {"value": value, "unit": "vectors/s", "cores": workers, "kind": "port",
                         "sample": f"{args.steps} full {n}x{m} RSR++ matvecs (C port of kernels.py:127-239)"},
        "e2e": {"value": value, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _metric(domain: str) -> str:
    return f"{domain} RSR++ matvec vectors/sec"


def _variants(args):
    if args.variant == "auto":
        return ["rsrpp", "rsr"] if args.config in BOTH_VARIANTS else ["rsrpp"]
    return ["rsrpp", "rsr"] if args.variant == "both" else [args.variant]


def _config_key(args, cfg, k):
    """The `config` object both arms print (identical keys and values for the same run)."""
    domain, n, m, desc = cfg
    return {"workload": desc, "n": n, "m": m, "k": k, "batch": BATCH.get(args.config, 1)}


def run_ours(args, cfg, dist=None, lite=False):
    """One measurement of `cfg`; returns the JSON line (dict).  lite: device timing only (no
    e2e, comparator or CPU legs) — the nested config-5 measurement of multi-GPU runs."""
    import torch
    import paper_2411_06360_b200 as rsr
    from paper_2411_06360_b200 import _native
    from paper_2411_06360_b200 import kernels as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    domain, n, m, desc = cfg
    # block width: the reference tuner (optimal_k_rsrpp) unless it differs from the measured B200
    # tuner (indexer.optimal_k_b200); results do not depend on k (integer products are exact)
    k_ref = rsr.optimal_k_rsrpp(n)
    k = args.k or rsr.optimal_k_b200(n, m)
    variants = _variants(args)

    # ---- data.  weak (default): rank g's shard = columns [g*m, (g+1)*m) of an n x (N*m) matrix.
    # strong (BASELINE config 5): rank g owns the column blocks [g*NB//N, (g+1)*NB//N) of ONE
    # n x m matrix (dist.shard_columns, the multiply_parallel partition), hash-generated per entry
    strong = args.config in STRONG
    m_full = m
    c0, c1 = (0, m)
    if strong:
        from paper_2411_06360_b200 import dist as D
        c0, c1 = D.shard_columns(m, k, world, rank)
        pad = max(D.slice_lengths(m, k, world))
        m = c1 - c0
        dA = hashed_ternary(n, c0, c1, m_full)
        A = dA.cpu().numpy()
    else:
        pad = m
        A = make_matrix(domain, n, m, seed=rank)
        dA = torch.from_numpy(A).cuda()
    fp32 = args.config in FP32
    v = (np.random.default_rng([0, n, 2]).standard_normal(n).astype(np.float32) if fp32 else make_vector(n))
    if domain == "ternary":  # first-use module loading of the preprocess kernels, untimed
        rsr.preprocess_ternary(dA[:256, :64].contiguous(), k if k <= 8 else 8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()  # preprocess only (the matrix is already in HBM)
    if domain == "ternary":
        idx = rsr.preprocess_ternary(dA, k)
    else:
        idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(A.astype(np.uint8)), k)
    torch.cuda.synchronize()
    preprocess_s = time.perf_counter() - t0

    # ---- the standard dense multiply on the GPU (csrc/dense.cu): comparator
    dense = rsr.DenseTernary(dA) if domain == "ternary" and not strong and not lite else None

    # ---- parity gate at full size (untimed): GPU keys + product vs the C oracle
    from oracle import c_oracle
    kp = c_oracle.keys_ternary(A, k, 1)
    kn = c_oracle.keys_ternary(A, k, -1) if domain == "ternary" else None
    halves = [idx.positive, idx.negative] if domain == "ternary" else [idx]
    for h, keys in zip(halves, [kp, kn]):
        if not np.array_equal(h.host_arrays()[2], keys):
            raise SystemExit("parity failure: device keys differ from the oracle")
    refs = {var: c_oracle.multiply_parallel(v.astype(np.float64), kp, kn, m, k, var != "rsr", cpu_threads())
            for var in variants}
    ref = refs[variants[0]]
    dv = torch.from_numpy(v).cuda()
    mult = rsr.multiply_ternary if domain == "ternary" else rsr.multiply_rsr

    def same(x, r=ref):
        x = np.asarray(x, np.float64)
        if fp32:
            return float(np.abs(x - r).max()) <= FP32_TOL * max(float(np.abs(r).max()), 1.0)
        return np.array_equal(x, r)
    for var in variants:
        if not same(mult(dv, idx, var).cpu().numpy(), refs[var]):
            raise SystemExit(f"parity failure: device {var} product differs from the oracle")
    del dA

    if args.config in BATCH:
        return run_batch(args, cfg, idx, A, v, kp, kn, k, k_ref, preprocess_s, world, rank, dist)

    # ---- index copies so consecutive steps never hit an index left in L2
    def clone_index(src):
        import copy
        from paper_2411_06360_b200.indexer import RsrIndex, TernaryIndex
        arrays = copy.copy(src.positive._arrays if domain == "ternary" else src._arrays)
        a0 = src.positive._arrays if domain == "ternary" else src._arrays
        arrays.perm = [t.clone() for t in a0.perm]
        arrays.seg = [t.clone() for t in a0.seg]
        arrays.bucket = [t.clone() for t in a0.bucket]
        arrays.desc = _native.IndexDesc.from_buffer_copy(a0.desc)
        for h in range(len(arrays.perm)):
            arrays.desc.half[h].perm = arrays.perm[h].data_ptr()
            arrays.desc.half[h].seg = arrays.seg[h].data_ptr()
            arrays.desc.half[h].bucket = arrays.bucket[h].data_ptr()
        if domain == "ternary":
            return TernaryIndex(RsrIndex(arrays, 0), RsrIndex(arrays, 1))
        return RsrIndex(arrays, 0)

    nblocks = idx.desc.nblocks
    hv = len(halves)
    row_stride = idx.desc.row_stride
    index_bytes = hv * nblocks * row_stride * 2 + 4 * n + 4 * m          # bucket u16 + v + out (scatter)
    canonical = hv * sum(2 * n + 4 * (1 << min(k, m - b * k)) for b in range(nblocks)) + 4 * n + 4 * m
    ncopies = max(2, -(-4 * L2_BYTES // (hv * nblocks * row_stride * 2)))
    copies = [idx] + [clone_index(idx) for _ in range(ncopies - 1)]
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    odt = torch.float32 if fp32 else torch.int32
    outs = [torch.zeros(pad, dtype=odt, device="cuda") for _ in range(2)]  # double-buffered slices
    gathered = [torch.empty(world * pad, dtype=odt, device="cuda") for _ in range(2)] if world > 1 else None
    comm = torch.cuda.Stream() if world > 1 else None
    peak, peak_kind = _peaks()

    def capture(var, mode, warm=False, indep=None):
        """K steps in one CUDA graph.  Step i multiplies index copy i % C into slice buffer
        i % 2; mode "overlap": the slice is all-gathered on the comm stream, which overlaps the
        next step's multiply (the multiply two steps later waits for that gather before reusing
        the buffer); "serial": the all-gather follows each multiply on the same stream; "none"."""
        fold = var != "rsr"
        indep = (args.launch == "independent") if indep is None else indep
        with_comm = mode == "overlap"
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        if with_comm:
            comm.wait_stream(stream)
        done = [None, None]
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                for i in range(args.steps):
                    b = i % 2
                    if done[b] is not None:
                        cap.wait_event(done[b])
                    K._multiply_device(dv, copies[0] if warm else copies[i % ncopies], fold, None, outs[b][:m],
                                       independent=indep)
                    if mode == "serial":
                        dist.all_gather_into_tensor(gathered[b], outs[b])
                    if with_comm:
                        ev = torch.cuda.Event()
                        ev.record(cap)
                        comm.wait_event(ev)
                        with torch.cuda.stream(comm):
                            dist.all_gather_into_tensor(gathered[b], outs[b])
                        done[b] = torch.cuda.Event()
                        done[b].record(comm)
                if with_comm:
                    cap.wait_stream(comm)  # the graph ends after the last gather
        stream.wait_stream(cap)
        g.replay()  # warm the graph itself
        torch.cuda.synchronize()
        return g

    def timed(graph):
        """R replays of the K-step graph (each bracketed by barrier + synchronize), clocks
        sampled during them; median replay.  Re-measured once if the clocks were bad."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.replays)]

        def region():
            with ClockSampler(local) as clocks:
                t_load = time.perf_counter() + 0.5
                while time.perf_counter() < t_load:  # load before the timed region (clocks settle)
                    graph.replay()
                    torch.cuda.synchronize()
                ms = []
                for e0, e1 in ev:
                    if world > 1:
                        dist.barrier()
                    torch.cuda.synchronize()
                    e0.record(stream)
                    graph.replay()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                t_load = time.perf_counter() + 0.2
                while time.perf_counter() < t_load:
                    graph.replay()
                    torch.cuda.synchronize()
            return ms, clocks.summary()
        ms, cs = region()
        remeasured = clocks_bad(cs)
        if remeasured:
            ms, cs = region()
        med = statistics.median(ms)
        if world > 1:  # max over ranks of the median replay
            tt = torch.tensor([med], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            med = float(tt.item())
        cs["remeasured"] = remeasured
        return med, ms, cs

    # warm-up steps (untimed) through the public device API
    for i in range(max(args.warmup, 3)):
        for var in variants:
            K._multiply_device(dv, copies[i % ncopies], var != "rsr", None, outs[0][:m])
    torch.cuda.synchronize()

    if world > 1:  # communicator warm-up on both streams (NCCL initialises lazily, never inside a capture)
        dist.all_gather_into_tensor(gathered[0], outs[0])
        with torch.cuda.stream(comm):
            dist.all_gather_into_tensor(gathered[1], outs[1])
        torch.cuda.synchronize()
    results = {}
    comm_mode, comm_error = ("overlap" if world > 1 else "none"), None
    for var in variants:
        g = None
        for mode in ([comm_mode, "serial"] if world > 1 else ["none"]):
            try:
                g = capture(var, mode)
                comm_mode = mode
                break
            except Exception as e:  # pragma: no cover - capture of the comm stream refused: serialise
                comm_error = repr(e)[:200]
                torch.cuda.synchronize()
        if g is None:
            raise SystemExit(f"graph capture failed: {comm_error}")
        med, ms, cs = timed(g)
        results[var] = (med, ms, cs)
        del g
        # the timed graph's own results (both slice buffers: the last two steps) against the oracle
        for b in range(min(2, args.steps)):
            got_b = outs[b][:m].double().cpu().numpy()
            ok = np.array_equal(got_b, refs[var]) if not fp32 else \
                float(np.abs(got_b - refs[var]).max()) <= FP32_TOL * max(1.0, float(np.abs(refs[var]).max()))
            if not ok:
                raise SystemExit(f"parity failure: the timed graph's step result ({var}, {args.launch}) differs")
    med, ms, clocks = results[variants[0]]
    ms_per_step = med / args.steps
    kernel_us = ms_per_step * 1e3 if world == 1 else None
    # weak: shard-matvecs per second (N shards per step); strong: full matvecs per second
    value = (1 if strong else world) * 1e3 / ms_per_step

    # SURVEY 8(d) "also report warm numbers": the same K steps on ONE index copy (L2-resident when
    # the index fits the 126 MB L2) — reported beside the cold value, never as it
    warm_us = None
    if world == 1 and not lite:
        g = capture(variants[0], "none", warm=True)
        wmed, _, _ = timed(g)
        del g
        warm_us = wmed / args.steps * 1e3
    # the other launch mode beside the headline (independent stream vs dependent chain)
    other_us = None
    if world == 1 and not lite:
        g = capture(variants[0], "none", indep=args.launch != "independent")
        omed, _, _ = timed(g)
        del g
        other_us = omed / args.steps * 1e3

    multi = None
    if world > 1:
        # compute-only (no all-gather) and the check of the gathered vector
        g = capture(variants[0], "none")
        cmed, _, _ = timed(g)
        del g
        kernel_us = cmed / args.steps * 1e3
        local_ref = torch.zeros(pad, dtype=torch.float64, device="cuda")
        local_ref[:m] = torch.from_numpy(ref).cuda()
        all_ref = torch.empty(world * pad, dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(all_ref, local_ref)
        K._multiply_device(dv, idx, variants[0] != "rsr", None, outs[0][:m])
        dist.all_gather_into_tensor(gathered[0], outs[0])
        torch.cuda.synchronize()
        ok = torch.equal(gathered[0].double(), all_ref) if not fp32 else \
            float((gathered[0].double() - all_ref).abs().max()) <= FP32_TOL * max(1.0, float(all_ref.abs().max()))
        okt = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if int(okt.item()) != 1:
            raise SystemExit("parity failure: the all-gathered vector differs from the ranks' oracle slices")
        multi = {"compute_only_us": cmed / args.steps * 1e3, "with_allgather_us": ms_per_step * 1e3,
                 "allgather_exposed_us": ms_per_step * 1e3 - cmed / args.steps * 1e3,
                 "allgather_bytes": world * pad * 4,
                 "overlap": ("all-gather of step i on a comm stream overlaps the multiply of step i+1 "
                             "(double-buffered slices; multiply grid capped at "
                             f"{os.environ.get('RSR_B200_MAX_CTAS', 'all')} CTAs so the collective has SMs)")
                            if comm_mode == "overlap" else
                            f"serialised all-gather after each multiply ({comm_error})",
                 "gathered_vector_check": "bitwise equal (int32) to the all-gathered per-rank C-oracle slices"
                 if not fp32 else "within 1e-5 norm-wise of the all-gathered per-rank C-oracle slices"}

    # ---- e2e through the reference-facing API with host buffers (rank-local)
    def e2e_time(vh, steps):
        # untimed: every copy's host session exists and has captured its call graph (a session
        # captures on its second publishing call)
        for i in range(max(3, 2 * ncopies + 1)):
            mult(vh, copies[i % ncopies])
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            res = mult(vh, copies[i % ncopies])
        e1.record(stream)
        torch.cuda.synchronize()
        if not same(res):
            raise SystemExit("parity failure on the e2e path")
        t = e0.elapsed_time(e1) / steps
        if world > 1:  # every rank's shard through the host API, max over ranks
            tt = torch.tensor([t], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    e2e_steps = 0 if lite else min(max(args.steps, 20), 500)
    scale = 1 if strong else world
    # csrc/host.cu: a single-split launch (rows <= 16384) pulls the 4-byte v from mapped host memory
    # itself and streams 8-byte seq-tagged result words back; larger ones: H2D, kernel, D2H of 4 * m
    pulls = n <= 16384
    d2h = (8 if pulls else 4) * m
    move = ("4-byte v pulled by the kernel from mapped host memory, results streamed back as tagged words"
            if pulls else "4-byte v over H2D, D2H of the results")
    if lite:
        e2e, extra_e2e = None, {}
    elif fp32:
        e2e_main_ms = e2e_time(v.copy(), e2e_steps)
        e2e = {"value": scale * 1e3 / e2e_main_ms, "unit": "vectors/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": d2h, "path": "rsr.multiply_ternary(numpy float32 v, idx)"}
        extra_e2e = {}
    else:
        v64 = v.astype(np.float64)  # the reference's calling convention (integer-valued fp64)
        e2e_main_ms = e2e_time(v64, e2e_steps)
        e2e_i32_ms = e2e_time(v.copy(), e2e_steps)
        e2e = {"value": scale * 1e3 / e2e_main_ms, "unit": "vectors/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": d2h,
               "path": f"rsr.{mult.__name__}(numpy float64 v, idx): the reference's calling convention; "
                       "integer values classified while staged (csrc/host_stage.cpp), int32 kernel (exact), "
                       + move + (" — on every rank's shard" if world > 1 else "")}
        extra_e2e = {"e2e_int32": {"value": scale * 1e3 / e2e_i32_ms, "unit": "vectors/s",
                                   "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": d2h,
                                   "path": f"rsr.{mult.__name__}(numpy int32 v, idx)"}}

    gpu_standard = None
    if dense is not None and not fp32 and int(np.abs(v).max()) <= 127:
        # the paper's standard multiply at its own roofline: the 2-bit matrix streamed once per
        # matvec with IDP4A on int8 activations (the reference's vectors are integers in
        # [-100, 100]); rotating copies of the 2-bit layout so every step reads HBM, like the index
        dv8 = dv.to(torch.int8)
        dout = dense.multiply_i8(dv8)
        if not same(dout.cpu().numpy()):
            raise SystemExit("parity failure: dense GPU product differs from the oracle")
        nq = max(2, -(-4 * L2_BYTES // dense.nbytes_i8))
        qcopies = [dense.q] + [dense.q.clone() for _ in range(nq - 1)]
        q0 = dense.q
        dg = torch.cuda.CUDAGraph()
        cap2 = torch.cuda.Stream()
        cap2.wait_stream(stream)
        dsteps = min(args.steps, 200)
        with torch.cuda.stream(cap2), torch.cuda.graph(dg, stream=cap2):
            for i in range(dsteps):
                dense.q = qcopies[i % nq]
                dense.multiply_i8(dv8, dout)
        dense.q = q0
        stream.wait_stream(cap2)
        dg.replay()
        torch.cuda.synchronize()
        dms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dg.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            dms.append(e0.elapsed_time(e1))
        d_us = statistics.median(dms) / dsteps * 1e3
        gpu_standard = {"value": 1e6 / d_us, "unit": "vectors/s", "kernel_us": d_us,
                        "weight_bytes": dense.nbytes_i8, "hbm_frac": dense.nbytes_i8 / (d_us * 1e-6) / 1e9 / peak,
                        "rsrpp_speedup": d_us / (ms_per_step * 1e3),
                        "l2": f"rotating {nq} copies of the 2-bit matrix (>= 4x L2)",
                        "what": "dense ternary GEMV on the same GPU (the paper's standard multiply): 2-bit matrix, "
                                "int8 activations, IDP4A (csrc/dense.cu dense_gemv_i8_kernel), exact int32"}
        del qcopies
        del dense

    def roof(var):
        # device time of the multiply alone (at N > 1: the compute-only graph of the main variant)
        us = kernel_us if (world > 1 and var == variants[0]) else results[var][0] / args.steps * 1e3
        achieved = canonical / (us * 1e-6) / 1e9
        prof = _profile(args.config, var)
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": prof.get("dram_bytes_per_launch"), "peak_kind": peak_kind,
                "algorithmic_bytes": canonical,
                "bytes_definition": "SURVEY.md 8(d) canonical: sum over halves, blocks of 2n + 4*2^w, + 4n + 4m",
                "index_bytes": index_bytes, "index_gbs": index_bytes / (us * 1e-6) / 1e9,
                "kernel_us": us, "traffic_source": prof.get("capture")}

    line = {
        "metric": _metric(domain),
        "value": value, "unit": "vectors/s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32" if fp32 else "int32", "data": "synthetic",
        "config": _config_key(args, cfg, k),
        "notes": {"k_tuner": f"optimal_k_b200 (the reference tuner gives k={k_ref}; results do not depend on k)",
                  "l2": f"rotating {ncopies} index copies (>= 4x L2): inputs larger than L2 every step",
                  "form": "scatter (fp32: exact two-limb fixed point)" if fp32 else "scatter (int32, exact)",
                  "variant": variants[0], "preprocess_s": round(preprocess_s, 4),
                  "launch": ("independent matvecs: each launch starts reducing on the SMs the previous one has "
                             "freed (RSR_MULTIPLY_INDEPENDENT; its output still waits for the previous launch)")
                  if args.launch == "independent" else "dependent chain: each launch waits for the previous one",
                  **({("dependent_chain_us" if args.launch == "independent" else "independent_us"): round(other_us, 3)}
                     if other_us is not None else {}),
                  **({"l2_warm_us": round(warm_us, 3),
                      "l2_warm_note": "one index copy replayed (L2-resident index when it fits): not the headline"}
                     if warm_us is not None else {}),
                  **({"value_unit": f"{n}x{m} shard-matvecs per second summed over {world} ranks (each step is "
                                    f"one matvec of the {n}x{world * m} matrix)"} if world > 1 and not strong else {}),
                  **({"shard_cols": [c0, c1], "matrix": "hash-generated per entry (same matrix for every N)"}
                     if strong else {})},
        "timing": {"replays": args.replays, "replays_ms": [round(x, 5) for x in ms], "statistic": "median replay",
                   "timed_region": f"{args.steps} steps in one CUDA graph"},
        "gpu_launches": args.steps * _count_launches(lambda: K._multiply_device(dv, idx, variants[0] != "rsr", None,
                                                                                outs[0][:m])),
        "e2e": e2e, **extra_e2e,
        "roofline": roof(variants[0]),
        "clocks": clocks,
    }
    if len(variants) > 1:
        line["variants"] = {var: {"kernel_us": results[var][0] / args.steps * 1e3,
                                  "value": (1 if strong else world) * 1e3 / (results[var][0] / args.steps),
                                  "roofline": roof(var), "replays_ms": [round(x, 5) for x in results[var][1]]}
                            for var in variants}
        line["variants"]["rsrpp_speedup_over_rsr"] = results["rsr"][0] / results["rsrpp"][0]
    if multi is not None:
        line["multi_gpu"] = multi
    if gpu_standard is not None:
        line["gpu_standard"] = gpu_standard
    if rank == 0 and world == 1 and not args.no_cpu and not lite:
        line["cpu_baseline"] = cpu_baseline(A, v, k_ref, domain, variants[0], args.cpu_seconds)
        if len(variants) > 1:
            line["cpu_baseline_rsr"] = cpu_baseline(A, v, k_ref, domain, "rsr", args.cpu_seconds / 2)
    if lite:
        line.pop("e2e", None)
    return line


def run_batch(args, cfg, idx, A, v, kp, kn, k, k_ref, preprocess_s, world, rank, dist):
    """BASELINE config 3: one step = rsr.multiply_batched of B vectors against one index."""
    import torch
    import paper_2411_06360_b200 as rsr
    from oracle import c_oracle
    domain, n, m, desc = cfg
    B = BATCH[args.config]
    rng = np.random.default_rng([0, n, B])
    Vh = rng.integers(-100, 101, size=(B, n)).astype(np.int32)
    V = torch.from_numpy(Vh).cuda()
    got = rsr.multiply_batched(V, idx).cpu().numpy()
    for i in (0, B // 2, B - 1):  # parity gate (untimed) on three of the vectors
        r = c_oracle.multiply_parallel(Vh[i].astype(np.float64), kp, kn, m, k, True, cpu_threads())
        if not np.array_equal(got[i].astype(np.float64), r):
            raise SystemExit("parity failure: batched product differs from the oracle")
    steps = args.steps
    for _ in range(max(args.warmup, 3)):
        rsr.multiply_batched(V, idx)  # the first call builds the batch plan (one-time, untimed)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    # the int32 batch path (batch plan + batch-native kernel) never synchronises: K batched
    # calls are captured in one CUDA graph like the single-vector configs
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        for _ in range(steps):
            outg = rsr.multiply_batched(V, idx)
    stream.wait_stream(cap)
    g.replay()
    torch.cuda.synchronize()
    if not np.array_equal(outg.cpu().numpy(), got):
        raise SystemExit("parity failure: captured batched product differs")

    def region():
        with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clocks:
            t_load = time.perf_counter() + 0.5
            while time.perf_counter() < t_load:
                g.replay()
                torch.cuda.synchronize()
            ms = []
            for _ in range(args.replays):
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0.record(stream)
                g.replay()
                t1.record(stream)
                torch.cuda.synchronize()
                ms.append(t0.elapsed_time(t1))
        return ms, clocks.summary()
    ms_list, cs = region()
    remeasured = clocks_bad(cs)
    if remeasured:
        ms_list, cs = region()
    cs["remeasured"] = remeasured
    ms = statistics.median(ms_list) / steps
    # e2e: pinned host V -> device, batched multiply, result -> host, every step
    Vp = torch.from_numpy(Vh).pin_memory()
    Oh = torch.empty((B, m), dtype=torch.int32).pin_memory()
    for _ in range(3):
        Oh.copy_(rsr.multiply_batched(Vp.cuda(non_blocking=True), idx), non_blocking=True)
    torch.cuda.synchronize()
    e_steps = min(steps, 50)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(e_steps):
        Oh.copy_(rsr.multiply_batched(Vp.cuda(non_blocking=True), idx), non_blocking=True)
        torch.cuda.current_stream().synchronize()
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / e_steps
    if not np.array_equal(Oh.numpy(), got):
        raise SystemExit("parity failure on the batched e2e path")
    nblocks = idx.desc.nblocks
    canonical = 2 * sum(2 * n + 4 * (1 << min(k, m - b * k)) for b in range(nblocks)) + B * (4 * n + 4 * m)
    adds = B * (2 * sum(n + 2 * (1 << min(k, m - b * k)) - 2 for b in range(nblocks)) + m)
    peak, peak_kind = _peaks()
    prof = _profile(args.config)
    line = {
        "metric": _metric(domain), "value": B * 1e3 / ms, "unit": "vectors/s",
        "n_gpus": world, "steps": steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": _config_key(args, cfg, k),
        "notes": {"k_tuner": f"optimal_k_b200 (the reference tuner gives k={k_ref})",
                  "form": "batch-native kernel (csrc/batch_lanes.cu): lanes span 64 vectors as packed int16 pairs, "
                          "9-wide re-cut batch plan with split slots, conflict-free shared-memory reductions",
                  "plan_extra_slots": int(idx._bplan[0].extra) if idx._bplan else None,
                  "preprocess_s": round(preprocess_s, 4)},
        "timing": {"replays": args.replays, "replays_ms": [round(x, 5) for x in ms_list],
                   "statistic": "median replay", "timed_region": f"{steps} batched calls in one CUDA graph"},
        "gpu_launches": None,
        "e2e": {"value": B * 1e3 / e2e_ms, "unit": "vectors/s", "h2d_bytes_per_step": 4 * B * n,
                "d2h_bytes_per_step": 4 * B * m, "path": "rsr.multiply_batched(pinned V.cuda(), idx) -> pinned host"},
        "roofline": {"bound": "hbm", "achieved": canonical / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": canonical / (ms * 1e-3) / 1e9 / peak, "traffic": prof.get("dram_bytes_per_launch"),
                     "peak_kind": peak_kind, "algorithmic_bytes": canonical,
                     "bytes_definition": "SURVEY.md 8(d) canonical, batch 64: index once + 64 x (4n + 4m)",
                     "adds_per_s": adds / (ms * 1e-3), "adds_frac": adds / (ms * 1e-3) / PEAK_ADDS,
                     "kernel_us": ms * 1e3},
        "clocks": cs,
    }
    line["gpu_launches"] = _count_launches(lambda: rsr.multiply_batched(V, idx)) * steps
    # the paper's standard multiply for a batch: dense int8 x int8 -> int32 GEMM on the tensor
    # cores (the library GEMM, cuBLASLt via torch._int_mm) against the int8 matrix
    try:
        A8 = torch.from_numpy(A).cuda()
        A8c = A8.t().contiguous().t()  # column-major operand for the int8 tensor-core GEMM
        del A8
        V8 = V.to(torch.int8)
        Y = torch._int_mm(V8, A8c)
        for i in (0, B - 1):
            r = c_oracle.multiply_parallel(Vh[i].astype(np.float64), kp, kn, m, k, True, cpu_threads())
            if not np.array_equal(Y[i].cpu().numpy().astype(np.float64), r):
                raise SystemExit("parity failure: dense int8 GEMM differs from the oracle")
        for _ in range(3):
            torch._int_mm(V8, A8c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            torch._int_mm(V8, A8c)
        e1.record(stream)
        torch.cuda.synchronize()
        g_us = e0.elapsed_time(e1) / 20 * 1e3
        line["gpu_standard"] = {"value": B * 1e6 / g_us, "unit": "vectors/s", "kernel_us": g_us,
                                "weight_bytes": int(A8c.numel()), "rsr_speedup": g_us / (ms * 1e3),
                                "what": "dense int8 GEMM on the tensor cores (cuBLASLt, torch._int_mm), exact int32; "
                                        "int8 matrix L2-resident only in part (268 MB)"}
        del A8c
    except RuntimeError as e:  # pragma: no cover - library shape limits
        line["gpu_standard"] = {"unavailable": str(e)[:200]}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(A, v, k_ref, domain, "rsrpp", args.cpu_seconds, batch=B)
    return line


def _count_launches(fn) -> int:
    """Kernels one call launches (torch profiler over one call)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        fn()
        torch.cuda.synchronize()
    return sum(1 for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA
               and "memset" not in e.name.lower() and "memcpy" not in e.name.lower())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--replays", type=int, default=11, help="timed replays of the K-step graph (median reported)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="ternary16384", choices=sorted(CONFIGS))
    ap.add_argument("--variant", default="auto", choices=["auto", "rsrpp", "rsr", "both"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--launch", default="independent", choices=["independent", "dependent"],
                    help="steps as independent matvecs (RSR_MULTIPLY_INDEPENDENT: a launch starts reducing on "
                         "SMs the previous one has freed) or as a dependent chain (each launch waits for the last)")
    ap.add_argument("--k", type=int, default=0, help="block width override (default: indexer.optimal_k_b200)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-strong", action="store_true", help="N > 1: skip the nested config-5 strong-scaling run")
    args = ap.parse_args()
    args.replays = max(1, args.replays)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # leave 4 SMs to the comm stream's all-gather (an NCCL kernel cannot start while the
        # persistent multiply grid holds every SM); 144 CTAs cost nothing at 16384^2 on one GPU
        # (22.39 vs 22.43 us: 1490 blocks take 11 rounds either way)
        os.environ.setdefault("RSR_B200_MAX_CTAS", "144")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = run_ours(args, cfg, dist)
    if world > 1 and args.config not in STRONG and not args.no_strong:
        # BASELINE config 5 beside the default weak-scaling line: ONE 65536^2 matrix column-sharded
        # over the ranks + all-gather (strong scaling), device timing only
        import copy
        a5 = copy.copy(args)
        a5.config, a5.steps, a5.variant = "ternary65536s", min(args.steps, 50), "rsrpp"
        try:
            l5 = run_ours(a5, CONFIGS["ternary65536s"], dist, lite=True)
            line["config5_strong"] = {key: l5.get(key) for key in
                                      ("value", "unit", "ms_per_step", "scaling", "config", "notes", "multi_gpu", "roofline")}
        except (Exception, SystemExit) as e:  # pragma: no cover - the main line stands on its own
            line["config5_strong"] = {"error": repr(e)[:300]}
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
