#!/usr/bin/env python3
"""Benchmark of the Balanced-Parallelism sparse gradient sync on B200.

Workload (BASELINE.json north_star target / configs[3]): a 1M x 64 fp32
embedding gradient per worker at 1% density (10,000 live rows of 64 non-zero
elements, integer values 1..16 so sums are exact), shared core omega = 0.5 of
the rows, the rest Zipf(1.05)-skewed over rows; n = N workers, one per GPU
(weak scaling: per-GPU work fixed).  One step = one full BP synchronisation:
extraction -> hierarchical hash + push -> aggregate + HashBitmap encode + pull
-> decode, dense gradients already in HBM.  Inputs (256 MB/GPU) exceed the
126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ... (one rank per GPU;
push/pull are NVLink stores into peer inboxes mapped with CUDA IPC).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse grad sync ms/iter (1/2/4/8 B200) + hash Mnnz/s as % HBM/NVLink roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--omega", type=float, default=0.5)
    ap.add_argument("--zipf", type=float, default=1.05)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--emulate", type=int, default=0,
                    help="extra: also time n emulated workers on one GPU (local mode)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the top-k / wire-format measurements (SURVEY §8f)")
    return ap.parse_args()


# --------------------------------------------------------------- workload ----

def live_rows(rows, per_worker, n, omega, zipf, seed):
    """Row ids per worker: a shared core of ceil(omega*z) rows + the remainder
    drawn without replacement from a Zipf(zipf) row popularity (ranks randomly
    permuted over row ids), Gumbel-top-k sampling, fixed seeds."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(rows)
    logw = np.empty(rows)
    logw[perm] = -zipf * np.log(np.arange(1, rows + 1))
    core_n = int(np.ceil(omega * per_worker))
    g = rng.gumbel(size=rows)
    core = np.argpartition(-(logw + g), core_n)[:core_n] if core_n else np.zeros(0, np.int64)
    out = []
    for w in range(n):
        r = np.random.default_rng(seed * 1000 + 17 + w)
        key = logw + r.gumbel(size=rows)
        key[core] = -np.inf
        rest = per_worker - core_n
        extra = np.argpartition(-key, rest)[:rest] if rest else np.zeros(0, np.int64)
        out.append(np.sort(np.concatenate([core, extra])))
    return out


def element_workload(m, n, density, omega, seed, hot_fraction=0.125, hot_mass=0.125,
                     workers=None):
    """Element-granular inputs with the reference generator's spec
    (zen::generate, zen/workload.hpp:22-30, 56-154): ceil(d*M) distinct
    indices per worker, a shared core of ceil(omega*d*M), the rest drawn per
    worker from a two-tier distribution (hot_mass of the draws in the first
    hot_fraction*M indices), integer values in [1, 16].  numpy streams, so the
    same spec, not the same bits as libstdc++'s mt19937_64 (the parity tests
    use the reference's own generator through oracle/_ref)."""
    z = int(np.ceil(density * m))
    hot = min(m, max(1, int(round(hot_fraction * m))))
    rng = np.random.default_rng(seed)

    def draw(k, used, r):
        out = np.empty(0, np.int64)
        while out.size < k:
            want = k - out.size
            nh = r.binomial(want, hot_mass if hot < m else 1.0)
            c = np.concatenate([r.integers(0, hot, nh), r.integers(hot, m, want - nh)]) \
                if hot < m else r.integers(0, hot, want)
            c = np.setdiff1d(np.unique(c), used, assume_unique=False)
            c = np.setdiff1d(c, out)
            out = np.concatenate([out, r.permutation(c)[:want]])
        return out

    core = draw(min(z, int(np.ceil(omega * density * m))), np.empty(0, np.int64), rng)
    res = {}
    for w in (range(n) if workers is None else workers):
        r = np.random.default_rng([seed, 0x10000 + w])
        rest = draw(z - core.size, core, r)
        idx = np.sort(np.concatenate([core, rest])).astype(np.uint64)
        res[w] = (idx, r.integers(1, 17, idx.size).astype(np.float32))
    return res


def dense_gradient(rows, width, live, seed):
    r = np.random.default_rng(seed)
    g = np.zeros((rows, width), np.float32)
    g[live] = r.integers(1, 17, (live.size, width)).astype(np.float32)
    return g.ravel()


# ----------------------------------------------------------------- clocks ----

class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line).  NVML is opened up front and polled
    in-process every ~2 ms (plus one synchronous sample at entry and exit), so
    even a timed region of a few ms has samples; nvidia-smi is the fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, {reasons})
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._bits = [nv.nvmlClocksEventReasonHwSlowdown,
                          nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwPowerCap]
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nv = nv
            self.source = "nvml"
        except Exception:
            self.source = "nvidia-smi"

    def _sample_nvml(self):
        nv = self._nv
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM), self._max,
                             {n for n, b in zip(self.NAMES, self._bits) if r & b}))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            f = [x.strip() for x in out.split(",")]
            if len(f) == 6 and f[0].replace(".", "").isdigit():
                self.samples.append((float(f[0]), float(f[1]),
                                     {n for n, v in zip(self.NAMES, f[2:]) if v.lower() == "active"}))
        except Exception:
            pass

    def _sample(self):
        try:
            self._sample_nvml() if self._nv else self._sample_smi()
        except Exception:
            pass

    def __enter__(self):
        self._sample()

        def run():
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(0.002 if self._nv else 0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": float(max(s[1] for s in self.samples)),
                "reasons": sorted(set().union(*[s[2] for s in self.samples])),
                "samples": len(self.samples), "source": self.source}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------ CPU baseline ----

def cpu_reference_step(args, n, dense_list, budget_s=12.0):
    """The reference's own CPU path (oracle/_ref: reference headers compiled in
    place): to_sparse of every worker + run_balanced_parallelism with a
    prebuilt table and lanes = host cores (n == 1: hierarchical_hash, the
    reference rejects n < 2).  Bounded sample: repeat until ~budget_s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import ref_oracle, COracle
    m = args.rows * args.width
    cores = os.cpu_count() or 1
    ro = ref_oracle()
    kind = "reference"
    if ro is None:  # never on a box that ran build(); kept for completeness
        kind = "port"
        co = COracle()
        t0 = time.perf_counter()
        ins = [co.to_sparse(d) for d in dense_list]
        if n >= 2:
            co.bp_sync(m, ins, seed=args.seed)
        dt = (time.perf_counter() - t0) * 1e3
        return {"value": dt, "unit": "ms/iter", "cores": 1, "kind": kind,
                "sample": f"1 step of the full workload, n={n}"}
    first = ro.bench_step(m, dense_list, lanes=cores, seed=args.seed, reps=1)
    step = first["to_sparse_ms"] + first["sync_ms"]
    reps = int(max(1, min(20, budget_s * 1e3 // max(step, 1.0))))
    res = ro.bench_step(m, dense_list, lanes=cores, seed=args.seed, reps=reps) if reps > 1 else first
    val = res["to_sparse_ms"] + res["sync_ms"]
    return {"value": round(val, 3), "unit": "ms/iter", "cores": cores, "kind": kind,
            "sample": (f"{reps + (1 if reps > 1 else 0)} full steps of the {args.rows}x{args.width} "
                       f"workload, n={n} workers simulated serially (to_sparse "
                       f"{res['to_sparse_ms']:.1f} ms + sync {res['sync_ms']:.1f} ms; one-time "
                       f"universe table {res['table_ms']:.0f} ms excluded)"),
            "stages_ms": {"to_sparse": round(res["to_sparse_ms"], 3),
                          "sync": round(res["sync_ms"], 3), "table_once": round(res["table_ms"], 1)}}


# --------------------------------------------------------------- exchange ----

NVLINK_PEER_GBPS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def exchange_report(ledger, n, stage_ms):
    """NVLink bytes each GPU sends in one sync and the rate they imply.  The
    push is fused into the scatter and the pull into the union/fold kernels,
    so the exchange has no kernel of its own: the rates below divide by the
    whole stage that carries it (a lower bound on the link rate)."""
    if n < 2:
        return {"note": "n = 1: no exchange"}
    # ledger bits use the reference widths: push 96 bits per COO entry, pull
    # B_s + 32 U_s; our wire sends u32 index + f32 value (64 bits) per entry
    push_out = ledger[0, 0] // 96 * 8
    pull_out = ledger[1, 0] // 8
    push_s = float(stage_ms[1]) * 1e-3
    pull_s = float(stage_ms[2]) * 1e-3
    pmax, qmax = float(push_out.max()), float(pull_out.max())
    return {"push_bytes_out_per_gpu_max": int(pmax), "pull_bytes_out_per_gpu_max": int(qmax),
            "push_GBps_lower_bound": round(pmax / push_s / 1e9, 1) if push_s else None,
            "pull_GBps_lower_bound": round(qmax / pull_s / 1e9, 1) if pull_s else None,
            "nvlink_peak_GBps": NVLINK_PEER_GBPS,
            "pull_frac_lower_bound": round(qmax / pull_s / 1e9 / NVLINK_PEER_GBPS, 4) if pull_s else None,
            "note": "push wire: u32 index + f32 value; pull: HashBitmap bits + f32 values to each "
                    "of the n-1 peers; rates = bytes / (hash_push | aggregate) stage time"}


# ------------------------------------------------------------ extras (f1/f2) ----

def compare_schemes(args, zen, d_dense, m, z, n, rank, stream, barrier, dist):
    """BP vs HC, ring centralization, AGsparse and OmniReduce-like on this
    run's gradients, one process per GPU: device time of K syncs (CUDA events, max over ranks); result
    indices checked equal to BP's on every rank."""
    import torch
    from paper_2309_13254_b200 import schemes as sch
    out = {}
    k = max(5, min(args.steps, 20))
    counts = None
    for name in ["hc", "ring", "agsparse", "omnireduce"]:
        if name in ("hc", "ring") and n & (n - 1):
            continue
        # create everywhere or nowhere: a rank that fails must not leave the
        # others waiting in the handle exchange
        try:
            sy = sch.HCSynchronizer(n, m, rank, max_nnz=int(z * 1.25) + 4096, scheme=name)
            okf = 1.0
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            sy, okf, err = None, 0.0, str(e)[:200]
        flag = torch.tensor([okf], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if float(flag[0]) < 1.0:
            out[name] = {"error": err if sy is None else "failed on another rank"}
            del sy
            continue
        sy.connect_process_group()
        for _ in range(3):
            sy.sync_dense(d_dense)
        sy.wait()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(k):
            sy.sync_dense(d_dense)
        a1.record(stream)
        barrier()
        sy.wait()
        t = torch.tensor([a0.elapsed_time(a1) / k], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        si, _ = sy.result()
        entry = {"ms": round(float(t[0]), 4), "result_nnz": int(si.numel())}
        if name == "hc":
            counts = sy.stage_bits()  # (index, value) bits sent per stage
        out[name] = entry
        del sy
    # densification ladder from rank 0's HC: state s covers ranks [0, 2^s)
    if counts is not None:
        nnz = torch.tensor([float(z)], device="cuda", dtype=torch.float64)
        alln = [torch.zeros_like(nnz) for _ in range(n)]
        dist.all_gather(alln, nnz)
        d = [float(x[0]) / float(m) for x in alln]
        union = [c[1] // 32 for c in counts] + [out["hc"]["result_nnz"]]  # |U_1|, |U_2|, ..
        gamma = {1: 1.0}
        kk = 2
        for u in union[1:]:
            gamma[kk] = (float(u) / float(m)) / (sum(d[:kk]) / float(kk))
            kk *= 2
        g = torch.tensor([gamma[kk] for kk in sorted(gamma)], device="cuda", dtype=torch.float64)
        dist.broadcast(g, 0)
        gamma = {kk: float(x) for kk, x in zip(sorted(gamma), g.cpu().numpy())}
        prof = sch.SparsityProfile(sum(d) / n, gamma, {})
        out["gamma"] = {str(kk): round(v, 4) for kk, v in gamma.items()}
        out["select_scheme"] = sch.select_scheme(prof, n)
        out["t_bp_coefficient"] = round(sch.t_bp_coefficient(n, gamma[n]), 4)
        out["t_hc_coefficient"] = round(sch.t_hc_coefficient(n, gamma), 4)
    return out


def measure_extras(args, zen, d_dense, peak, reps=10):
    """The components either side of the sync: top-k
    sparsification of the dense gradient (f2) and the COO / tensor-block wire
    formats of its sparse form (f1), each a synchronous C-ABI call on
    device-resident data, timed with CUDA events; the reference's CPU path on
    a bounded sample beside it."""
    import ctypes as C
    import torch
    lib = zen.load()
    ctx = zen.context()
    ctx.bind_stream()
    stream = torch.cuda.current_stream()
    m = d_dense.numel()
    out = {}
    frac = args.density
    keep = min(m, int(np.ceil(frac * m)))
    oi = torch.empty(keep, dtype=torch.int64, device="cuda")
    ov = torch.empty(keep, dtype=torch.float32, device="cuda")
    got = C.c_uint64()

    def topk():
        rc = lib.zen_sparsify_topk(ctx.h, C.c_void_p(d_dense.data_ptr()), m, frac,
                                   C.c_void_p(oi.data_ptr()), C.c_void_p(ov.data_ptr()), keep,
                                   C.byref(got))
        assert rc == 0, lib.zen_last_error_message()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t = timed(topk)
    one_pass = 4 * m + 12 * got.value
    out["sparsify_topk"] = {
        "fraction": frac, "kept": int(got.value), "ms_per_call": round(t, 4),
        "hbm_frac_of_one_pass": round(one_pass / (t * 1e-3) / 1e9 / peak, 4),
        "note": "radix select: 2 HBM passes over the dense input (histogram, bucket-floor tile pass); frac vs a single 4M-byte read"}
    # the wire formats of the extracted sparse gradient
    nz = torch.nonzero(d_dense).flatten()
    vals = d_dense[nz].contiguous()
    cnt = nz.numel()
    for name, f in [("coo64", zen.WireFormat.coo()), ("tensor_block256", zen.WireFormat.tensor_block())]:
        fc = f._c()
        info = zen._lib.MessageInfoC()
        lib.zen_encode(ctx.h, C.byref(fc), None, 0, C.c_void_p(nz.data_ptr()),
                       C.c_void_p(vals.data_ptr()), cnt, m, None, 0, C.byref(info))
        pay = torch.empty(max(int(info.payload_bytes), 1), dtype=torch.uint8, device="cuda")
        di = torch.empty(cnt, dtype=torch.int64, device="cuda")
        dv = torch.empty(cnt, dtype=torch.float32, device="cuda")
        n2 = C.c_uint64()

        def enc():
            assert lib.zen_encode(ctx.h, C.byref(fc), None, 0, C.c_void_p(nz.data_ptr()),
                                  C.c_void_p(vals.data_ptr()), cnt, m, C.c_void_p(pay.data_ptr()),
                                  int(info.payload_bytes), C.byref(info)) == 0

        def dec():
            assert lib.zen_decode(ctx.h, C.byref(fc), None, 0, C.byref(info),
                                  C.c_void_p(pay.data_ptr()), C.c_void_p(di.data_ptr()),
                                  C.c_void_p(dv.data_ptr()), cnt, C.byref(n2)) == 0
        te, td = timed(enc), timed(dec)
        out[name] = {"entries": cnt, "payload_bytes": int(info.payload_bytes),
                     "encode_ms": round(te, 4), "decode_ms": round(td, 4),
                     "encode_GBps": round(info.payload_bytes / (te * 1e-3) / 1e9, 1),
                     "decode_GBps": round(info.payload_bytes / (td * 1e-3) / 1e9, 1)}
    # the reference's CPU sparsify_topk on a bounded sample (a 4M-element prefix)
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import ref_oracle
        ro = ref_oracle()
        if ro is not None:
            sample = d_dense[: 1 << 22].cpu().numpy()
            t0 = time.perf_counter()
            ro.sparsify_topk(sample, frac)
            dt = (time.perf_counter() - t0) * 1e3
            out["sparsify_topk"]["cpu_reference"] = {
                "ms": round(dt, 2), "cores": 1, "kind": "reference",
                "sample": f"4,194,304-element prefix of the dense gradient (x{m / (1 << 22):.1f} "
                          f"for the full tensor: ~{dt * m / (1 << 22):.0f} ms)"}
    except Exception as e:  # the CPU sample is informational
        out["sparsify_topk"]["cpu_reference"] = {"error": str(e)[:200]}
    return out


# --------------------------------------------------------------- our arm ----

def config_dict(args, n, z):
    return {"workload": f"embedding gradient {args.rows}x{args.width} fp32, {args.density:.2%} "
                        f"density per worker (row-structured, omega={args.omega}, "
                        f"Zipf({args.zipf}) rows), n={n} workers (1 per GPU), BP sync",
            "rows": args.rows, "width": args.width, "universe": args.rows * args.width,
            "nnz_per_worker": z, "n_workers": n, "hash": {"k": 3, "r1_multiplier": 2.0,
                                                          "r2_ratio": 0.1, "seed": args.seed},
            "l2": "inputs larger than L2 (256 MB dense fp32 per GPU > 126 MB L2); no flush",
            "parallelism": f"dp{n}"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(args.gpus, world)
    m = args.rows * args.width
    per_worker_rows = int(np.ceil(args.density * args.rows))
    z = per_worker_rows * args.width

    if args.impl == "reference":
        if rank != 0:
            return 0
        rows = live_rows(args.rows, per_worker_rows, n, args.omega, args.zipf, args.seed)
        dense = [dense_gradient(args.rows, args.width, rows[w], args.seed + w) for w in range(n)]
        vals = []
        base = cpu_reference_step(args, n, dense, budget_s=2.0)
        k = max(1, args.steps)
        for _ in range(min(k, 5)):
            vals.append(cpu_reference_step(args, n, dense, budget_s=0.0)["value"])
        v = float(np.median(vals))
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms/iter",
                "n_gpus": args.gpus, "steps": len(vals), "warmup": 1, "ms_per_step": round(v, 3),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": config_dict(args, n, z),
                "cpu_baseline": {"value": round(v, 3), "unit": "ms/iter", "cores": base["cores"],
                                 "kind": base["kind"], "sample": base["sample"]},
                "e2e": {"value": round(v, 3), "unit": "ms/iter", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    torch.cuda.set_device(local_rank)
    torch.cuda.set_stream(torch.cuda.Stream())  # non-legacy stream: the sync is graph-replayed
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_2309_13254_b200 as zen

    rows = live_rows(args.rows, per_worker_rows, n, args.omega, args.zipf, args.seed)
    host = dense_gradient(args.rows, args.width, rows[rank], args.seed + rank)
    d_dense = torch.from_numpy(host).cuda()
    params = zen.HashParams(seed=args.seed)
    bp = zen.BPSynchronizer(n, m, max_nnz=int(z * 1.25) + 4096, params=params,
                            rank=None if n == 1 else rank)
    if n > 1:
        bp.connect_process_group()
    stream = torch.cuda.current_stream()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        bp.sync_dense([d_dense])
    bp.wait()
    # correctness guard on the benchmarked configuration (cheap identity checks)
    cnt = bp.result_count()
    assert cnt >= z and cnt <= n * z, f"result size {cnt} out of range"
    launches0 = zen.load().zen_kernel_launches()
    with ClockSampler(local_rank) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # the barrier right before the first event: the sampler's start-up
        # (NVML calls) must not skew the ranks' start times
        barrier()
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            bp.sync_dense([d_dense])
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        e1.record(stream)
        barrier()
    launches = zen.load().zen_kernel_launches() - launches0
    bp.wait()
    ms = e0.elapsed_time(e1) / args.steps
    # stage breakdown: a second pass of the same K syncs replayed from the graph
    # variant with CUDA-event nodes between the stages (the nodes cost a few us
    # each, so the headline `value` above is timed without them)
    bp.stage_times()  # reset
    bp.enable_timing(True)
    for _ in range(2):
        bp.sync_dense([d_dense])
    bp.wait()
    bp.stage_times()
    barrier()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        bp.sync_dense([d_dense])
    s1.record(stream)
    barrier()
    bp.wait()
    staged_ms = s0.elapsed_time(s1) / args.steps
    stage_ms, timed = bp.stage_times()
    bp.enable_timing(False)
    stage_ms = stage_ms / max(timed, 1)
    # the roofline kernel alone: back-to-back launches, CUDA events on its stream
    ext_kernel_ms = bp.time_extract(d_dense, iters=max(20, args.steps // 4))
    per_rank = None
    if dist:
        t = torch.tensor([ms, host_ms, staged_ms] + list(stage_ms), device="cuda",
                         dtype=torch.float64)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        allt = torch.stack(allt).cpu().numpy()
        per_rank = [{"ms": round(float(r[0]), 4), "host_enqueue_ms": round(float(r[1]), 4),
                     "stage_ms": [round(float(x), 4) for x in r[3:]]} for r in allt]
        ms, host_ms, staged_ms = (float(allt[:, i].max()) for i in range(3))
        stage_ms = allt[:, 3:].max(0)
    ledger, counts, agg = bp.ledger()
    union = int(bp.result_count())

    # e2e: host (pinned) dense -> H2D -> sync -> D2H result, through the C-ABI
    e2e = None
    if not args.no_e2e:
        pin = torch.from_numpy(host).pin_memory()
        cap = n * z + 16
        oi = torch.empty(cap, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        ov = torch.empty(cap, dtype=torch.float32).pin_memory().numpy()
        hd = [pin.numpy()]
        bp.sync_host(hd, oi, ov)
        barrier()
        k2 = max(3, min(args.steps, 10))
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(k2):
            got = bp.sync_host(hd, oi, ov)
        t1.record(stream)
        barrier()
        e2e_ms = t0.elapsed_time(t1) / k2
        if dist:
            t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        e2e = {"value": round(e2e_ms, 4), "unit": "ms/iter", "h2d_bytes_per_step": 4 * m * n,
               "d2h_bytes_per_step": 12 * got * n,
               "path": "zen_bp_sync_host (C-ABI): pinned host dense -> device -> host result"}

    # the paper's comparison at N > 1: the same
    # gradients through Hierarchical Centralization, ring centralization and
    # AGsparse in rank mode, and select_scheme's choice from the measured
    # densification ladder (rank 0's HC stage counts are the prefix unions)
    schemes = None
    if dist and not args.no_extras:
        try:
            schemes = compare_schemes(args, zen, d_dense, m, z, n, rank, stream, barrier, dist)
        except Exception as e:  # noqa: BLE001 -- the headline line must still print
            schemes = {"error": str(e)[:300]}

    # extra: n workers emulated on one GPU (local mode), e.g. the 8-worker headline
    emu = None
    if args.emulate and rank == 0 and world == 1:
        ne = args.emulate
        rows_e = live_rows(args.rows, per_worker_rows, ne, args.omega, args.zipf, args.seed)
        dd = [torch.from_numpy(dense_gradient(args.rows, args.width, rows_e[w], args.seed + w)).cuda()
              for w in range(ne)]
        be = zen.BPSynchronizer(ne, m, max_nnz=int(z * 1.25) + 4096, params=params)
        for _ in range(3):
            be.sync_dense(dd)
        be.wait()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ke = max(3, args.steps // 2)
        for _ in range(ke):
            be.sync_dense(dd)
        a1.record(stream)
        torch.cuda.synchronize()
        be.wait()
        be.enable_timing(True)  # stage breakdown from a second pass
        for _ in range(ke):
            be.sync_dense(dd)
        be.wait()
        sms, kk = be.stage_times()
        be.enable_timing(False)
        nzr = np.zeros(args.rows, bool)
        for w in range(ne):
            nzr[rows_e[w]] = True
        union = be.result_count()
        emu = {"workers": ne, "ms_per_sync_one_gpu": round(a0.elapsed_time(a1) / ke, 4),
               "stage_ms": {nm: round(float(x) / max(kk, 1), 4)
                            for nm, x in zip(zen.STAGE_NAMES, sms)},
               "union": union, "union_ok": bool(union == int(nzr.sum()) * args.width)}
        del be, dd

    # the same sync on element-granular gradients (the reference generator's
    # spec, zen/workload.hpp:123-154): one non-zero per position instead of
    # whole 64-float rows, the harder case for the bitmap fold and decode
    elem = None
    if not args.no_extras:
        ei, evv = element_workload(m, n, args.density, args.omega, args.seed + 17,
                                   workers=[rank])[rank]
        ed = torch.zeros(m, dtype=torch.float32, device="cuda")
        ed[torch.from_numpy(ei.view(np.int64)).cuda()] = torch.from_numpy(evv).cuda()
        be = zen.BPSynchronizer(n, m, max_nnz=int(ei.size * 1.25) + 4096, params=params,
                                rank=None if n == 1 else rank)
        if n > 1:
            be.connect_process_group()
        for _ in range(max(3, args.warmup)):
            be.sync_dense([ed])
        be.wait()
        barrier()
        x0 = torch.cuda.Event(enable_timing=True)
        x1 = torch.cuda.Event(enable_timing=True)
        kx = max(5, args.steps // 2)
        x0.record(stream)
        for _ in range(kx):
            be.sync_dense([ed])
        x1.record(stream)
        barrier()
        be.wait()
        ems = x0.elapsed_time(x1) / kx
        be.enable_timing(True)
        for _ in range(kx):
            be.sync_dense([ed])
        be.wait()
        esm, ek = be.stage_times()
        be.enable_timing(False)
        if dist:
            t = torch.tensor([ems] + list(esm / max(ek, 1)), device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems, esm, ek = float(t[0]), t[1:].cpu().numpy(), 1
        elem = {"workload": f"element-granular {m} positions, {args.density:.2%} density, "
                            f"omega={args.omega}, two-tier (1/8 hot, 1/8 mass)",
                "nnz_per_worker": int(ei.size), "ms_per_sync": round(ems, 4),
                "union_nnz": int(be.result_count()),
                "stage_ms": {nm: round(float(x) / max(ek, 1), 5)
                             for nm, x in zip(zen.STAGE_NAMES, esm)}}
        del be, ed

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel (extraction: streams the 256 MB dense gradient)
    peak, peak_src = measured_peaks()
    ext_ms = float(ext_kernel_ms)
    alg_bytes = 4 * m + 12 * z  # 4M + E*z, E = 12 B (u64 index + f32 value)
    achieved = alg_bytes / (ext_ms * 1e-3) / 1e9 if ext_ms > 0 else None
    traffic = ncu_traffic().get("k_extract")
    roofline = {"kernel": "k_extract (non-zero extraction, HBM-bound)", "bound": "hbm",
                "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": traffic, "algorithmic_bytes_per_launch": alg_bytes,
                "peak_source": peak_src,
                "launch_ms": round(ext_ms, 5),
                "timing": "k_extract_tiles alone, back-to-back launches, CUDA events on its stream "
                          "(zen_bp_time_extract); in-sync stage time in stage_ms.extract"}
    hash_ms = float(stage_ms[1])
    hash_bytes = 24 * z  # 2*E*z
    total_nnz = n * z
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/iter", "n_gpus": n,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (row-structured embedding gradients, integer values)",
        "config": config_dict(args, n, z),
        "throughput_mnnz_per_s": round(total_nnz / (ms * 1e-3) / 1e6, 1),
        "stage_ms": {nm: round(float(x), 5) for nm, x in zip(zen.STAGE_NAMES, stage_ms)},
        "stage_pass_ms_per_step": round(staged_ms, 4),
        "hash_stage": {"mnnz_per_s": round(z / (hash_ms * 1e-3) / 1e6, 1) if hash_ms else None,
                       "algorithmic_bytes": hash_bytes,
                       "hbm_frac": round(hash_bytes / (hash_ms * 1e-3) / 1e9 / peak, 4) if hash_ms else None,
                       "note": "includes the fused NVLink push (scatter into owner inboxes)"},
        "exchange": exchange_report(ledger, n, stage_ms),
        "host_enqueue_ms_per_step": round(host_ms, 4),
        "union_nnz": union, "gpu_launches": int(launches),
        "kernels_per_sync": bp.kernels_per_sync(),
        "roofline": roofline,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if per_rank:
        line["per_rank"] = per_rank
    if emu:
        line["emulated_local"] = emu
    if elem:
        line["element_granular"] = elem
    if world == 1 and not args.no_extras:
        line["extras"] = measure_extras(args, zen, d_dense, peak)
    if schemes is not None:
        line["schemes"] = dict(schemes, bp_ms=round(ms, 4),
                               note="rank mode, same gradients; CUDA events, max over ranks")
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_reference_step(args, n, [host])
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
