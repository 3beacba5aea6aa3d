"""Benchmark of the TTTP + sparse-MTTKRP hot path (BASELINE.json metric).

Workload (BASELINE cfg 2, the configuration the metric is quoted on): sparse
order-3 fp64 tensor 10,000^3 with 1e7 uniform distinct nonzeros, values
N(0,1), int32 indices, R = 16 factors N(0, 1/R).  One *step* = one TTTP plus
one sparse MTTKRP on each of the three modes.  ``value`` = nonzeros processed
per second per kernel pass, i.e. 4 * nnz / step time, with inputs resident in
HBM (device-resident factors/values, pattern built once = the reference's
cached coords / mode groups).  ``e2e`` = the same metric through the public
drop-in API with host (numpy, pinned) values and factors, host<->device copies
inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (launched by torchrun, one rank per GPU, NCCL): weak scaling -- every
rank owns a distinct 1e7-nonzero shard of one N x 1e7-nonzero tensor over the
same index space; TTTP is local, the per-mode MTTKRP partial outputs (I_n x R)
are summed with an NCCL all-reduce (the real exchange step of a
nonzero-partitioned MTTKRP).  Time = max over ranks of device time.

``--impl reference`` times the reference's CPU algorithm (the C restatement
in oracle/, OpenMP over all host threads, restating the numba prange loops of
_jit.py) on the same workload, on rank 0 only.
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

HBM_FALLBACK_GBS = 6650.0
R = 16
NNZ = 10_000_000


def num_sms_probe(torch):
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (NVML / nvidia-smi during the timed region)

REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.  NVML
    (nvidia-ml-py) polled from a thread every ~2 ms, so even a 40 ms region
    gets many samples; ``nvidia-smi -lms 50`` if NVML is unavailable."""

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []  # (time, sm_mhz, max_mhz, reasons)
        self.marks = []
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        cmd = ["nvidia-smi", f"--id={self.index}",
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
               "--format=csv,noheader,nounits", "-lms", "50"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read_smi, daemon=True)
        self.t.start()
        t_end = time.perf_counter() + 10.0
        while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
            time.sleep(0.02)

    def _poll_nvml(self):
        pynvml, h = self.nvml
        while not self._stop.is_set():
            try:
                sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                r = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception:
                return
            self.lines.append((time.perf_counter(), sm, self.max_mhz, r))
            time.sleep(0.002)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                r = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
                self.lines.append((time.perf_counter(), float(parts[0]), float(parts[1]), r))
            except (ValueError, IndexError):
                continue

    def mark(self, tag):
        self.marks.append((tag, time.perf_counter()))

    def stop(self):
        self._stop.set()
        if self.proc is None and self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        t0 = dict(self.marks).get("start", 0.0)
        t1 = dict(self.marks).get("stop", time.perf_counter())
        window = [x for x in self.lines if t0 <= x[0] <= t1]
        if not window:  # region shorter than the sampling period: nearest samples
            window = sorted(self.lines, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))[:2]
        reasons = 0
        for x in window:
            reasons |= x[3]
        names = [n for bit, n in REASON_BITS.items() if reasons & bit and n != "gpu_idle"]
        sm = [x[1] for x in window]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(x[2] for x in window) if window else None,
                "reasons": names, "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------

def algorithmic_bytes(order, nnz, rank, dims, vbytes=8, ibytes=4):
    """gather-inclusive bytes per launch."""
    tttp = nnz * (order * ibytes + 2 * vbytes + order * rank * vbytes)
    mtt = [nnz * (order * ibytes + vbytes + (order - 1) * rank * vbytes) + dims[n] * rank * vbytes
           for n in range(order)]
    compulsory = nnz * (order * ibytes + 2 * vbytes) + sum(dims) * rank * vbytes
    return tttp, mtt, compulsory


def compulsory_bytes(order, nnz, rank, dims, vbytes=8, ibytes=4):
    """SURVEY.md 8(d) compulsory bytes per launch: the nonzero stream plus every
    factor / output row touched once (what HBM must deliver at least).
    TTTP: m (N s_i + 2 s_v) + sum_k I_k R s_v; MTTKRP mode n: m (N s_i + s_v)
    + sum_k I_k R s_v (the output I_n x R included)."""
    facs = sum(dims) * rank * vbytes
    tttp = nnz * (order * ibytes + 2 * vbytes) + facs
    mtt = nnz * (order * ibytes + vbytes) + facs
    return tttp, mtt


def nccl_summary(path, world):
    """Rank 0's NCCL INIT log (NCCL_DEBUG=INFO): version, communicator sizes,
    NVLS (NVSwitch multicast / in-switch reduction) availability."""
    import re
    try:
        text = open(path).read()
    except (OSError, TypeError):
        return {"log": None}
    sizes = sorted({int(x) for x in re.findall(r"nRanks (\d+)", text)})
    ver = re.search(r"NCCL version ([0-9.]+)", text)
    return {"log": path, "lines": text.count("\n"), "version": ver.group(1) if ver else None,
            "comm_nranks": sizes, "comm_nranks_ok": world in sizes,
            "nvls": bool(re.search(r"NVLS multicast support is available|NVLS comm", text))}


def run_reference(args):
    """CPU arm: the reference algorithm (oracle C restatement), all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1910_02371_b200 import synth
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    shape, keys, values, factors = synth.cfg2()
    t = O.OTensor(shape, keys, values)
    for mode in range(3):  # warm caches like the reference's cached coords/groups
        t.mode_group(mode)

    def step():
        O.tttp(t, factors)
        for mode in range(3):
            O.mttkrp(t, factors, mode)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = 4 * t.nnz / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE cfg 2 shape/value laws)",
        # same config block as the GPU arm (the same synth.cfg2() tensor, seed 2);
        # with --gpus N the GPU arm shards this one tensor by nonzero ranges
        "config": dict(CONFIG, parallelism=f"nnz-shard{args.gpus}" if args.gpus > 1 else "1gpu"),
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": "port",
                         "sample": f"full cfg 2 workload, {args.steps} steps after "
                                   f"{args.warmup} warm-up (oracle/cpfit_oracle.c, OpenMP)"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "nonzeros/sec for TTTP & MTTKRP (TTTP + MTTKRP all modes, per kernel pass)"
CONFIG = {"workload": "BASELINE cfg 2: sparse 10000^3, 1e7 uniform distinct nnz, R=16, fp64; "
                      "step = TTTP + MTTKRP modes 0,1,2",
          "nnz_per_gpu": NNZ, "rank": R, "shape": [10000, 10000, 10000],
          "l2": "inputs larger than L2 (0.28 GB index+value stream per pass > 126 MB); "
                "factors (3.84 MB) L2-resident by design"}


def cpu_baseline_sample(seconds=12.0):
    from oracle import oracle as O
    from paper_1910_02371_b200 import synth
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    shape, keys, values, factors = synth.cfg2()
    t = O.OTensor(shape, keys, values)
    for mode in range(3):
        t.mode_group(mode)
    O.tttp(t, factors)
    O.mttkrp(t, factors, 0)  # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        O.tttp(t, factors)
        for mode in range(3):
            O.mttkrp(t, factors, mode)
        n += 1
        if time.perf_counter() - t0 > seconds or n >= 50:
            break
    dt = (time.perf_counter() - t0) / n
    return {"value": 4 * t.nnz / dt, "unit": "nnz/s", "cores": threads, "kind": "port",
            "sample": f"{n} full cfg-2 steps (TTTP + 3 MTTKRP, 1e7 nnz) with "
                      "oracle/cpfit_oracle.c on all host threads"}


def cpu_info():
    """Host cores used by the CPU legs and the CPU model (this box)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cores": os.cpu_count() or 1, "model": model}


def als_section(world, rank, dev, sweeps=3, cpu=True):
    """BASELINE cfg 3 (480,189 x 17,770 x 2,182, 100,480,507 Zipf nnz, R=32,
    lambda=1e-5): device-generated seeded instance; ALS sweep time at N GPUs
    (row-sharded with an NCCL all-gather per mode when N > 1; strong scaling),
    plus one CCD++ sweep on a single GPU."""
    import torch
    import torch.distributed as dist

    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import synth
    from paper_1910_02371_b200.optim import _als_ls_device, _ccd_ls_device
    R3, REG = 32, 1e-5
    t0 = time.perf_counter()
    shape, keys, vals = synth.cfg3_device()
    gen_s = time.perf_counter() - t0
    g = cp.RngState(0).child(0).generator()
    init = [torch.from_numpy(g.random((d, R3)) / np.sqrt(R3)).to(dev) for d in shape]
    stream = torch.cuda.current_stream()
    out = {"workload": "BASELINE cfg 3 shape/nnz: 480189x17770x2182, 100480507 nnz, modes 0/1 "
                       "Zipf(1), mode 2 uniform, values 1..5; R=32, lambda=1e-5 (direct solve)",
           "generation_s": gen_s, "n_gpus": world}
    if world == 1:
        t = cp.SparseTensor.from_device(shape, keys, vals)
        del keys
        F = [f.clone() for f in init]
        t1 = time.perf_counter()
        _als_ls_device(t, F, REG)  # warm-up sweep: builds the mode layouts
        torch.cuda.synchronize()
        out["first_sweep_incl_layout_s"] = time.perf_counter() - t1
        _als_ls_device(t, F, REG)  # second warm-up: allocator caches settle
        times = []
        for _ in range(sweeps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _als_ls_device(t, F, REG)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        out["als_sweep_ms"] = float(np.median(times))
        out["als_sweep_ms_all"] = times
        # per-phase split of one more sweep (MTTKRP rhs vs Gram + solve)
        from paper_1910_02371_b200.optim import _als_mode_device
        phases = []
        for mode in range(3):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record(stream)
            F[mode] = _als_mode_device(t, F, mode, REG)
            e[1].record(stream)
            torch.cuda.synchronize()
            phases.append(e[0].elapsed_time(e[1]))
        out["als_mode_update_ms"] = phases
        from paper_1910_02371_b200.losses import ls_data_term
        out["rmse_after"] = float(np.sqrt(ls_data_term(t, F) / t.nnz))
        # "ALS completion with implicit CG" (BASELINE cfg 3): the Gram-free
        # per-row CG update (cpfit_gram_matvec), four sweeps from the same init
        # as the direct sweeps (each mode warm-started from its current rows)
        from paper_1910_02371_b200.optim import _als_ls_cg_device
        Fc = [f.clone() for f in init]
        cg_tol, cg_max = 5e-3, min(30, 3 * R3)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base_mem = torch.cuda.memory_allocated()
        cg_ms, cg_it = [], []
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, its = _als_ls_cg_device(t, Fc, REG, cg_tol, cg_max)
            b.record(stream)
            torch.cuda.synchronize()
            cg_ms.append(a.elapsed_time(b))
            cg_it.append(its)
        out["als_cg"] = {
            "sweep_ms": cg_ms[-1], "sweep_ms_all": cg_ms, "cg_iters_per_mode": cg_it, "cg_tol": cg_tol,
            "cg_max": cg_max, "rmse_after": float(np.sqrt(ls_data_term(t, Fc) / t.nnz)),
            "peak_extra_GB": (torch.cuda.max_memory_allocated() - base_mem) / 1e9,
            "what": "SolverConfig(als_solver='cg'): per-row CG on (G_i + lambda I) x_i = rhs_i with "
                    "G_i p_i from one pass over the nonzeros (no I x R x R Gram buffer: the direct "
                    "sweep allocates 3.9 GB for mode 0); rows stop at ||r_i|| <= cg_tol ||b_i|| and "
                    "are skipped by later passes; four sweeps from the direct sweeps' init"}
        del Fc
        F = [f.clone() for f in init]
        _ccd_ls_device(t, F, REG)  # warm-up: the per-mode rhat copies' allocations
        ccd_ms = []
        for _ in range(3):
            F = [f.clone() for f in init]
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _ccd_ls_device(t, F, REG)
            b.record(stream)
            torch.cuda.synchronize()
            ccd_ms.append(a.elapsed_time(b))
        out["ccd_sweep_ms"] = float(np.median(ccd_ms))
        out["ccd_sweep_ms_all"] = ccd_ms
        # one Gauss-Newton step from the ALS iterate
        from paper_1910_02371_b200.optim import CompletionState, SolverConfig
        from paper_1910_02371_b200.second_order import gn_step_device
        from paper_1910_02371_b200.losses import get_loss
        gcfg = SolverConfig(rank=R3, reg=REG, gn_damping=1.0)
        st = CompletionState(factors=F, rng=cp.RngState(0))
        Fg = [f.clone() for f in init]
        _als_ls_device(t, Fg, REG)
        gn_step_device(t, Fg, get_loss("ls"), gcfg, st, "gauss_newton")  # warm-up
        st = CompletionState(factors=F, rng=cp.RngState(0))
        Fg = [f.clone() for f in init]
        _als_ls_device(t, Fg, REG)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        cg = gn_step_device(t, Fg, get_loss("ls"), gcfg, st, "gauss_newton")
        b.record(stream)
        torch.cuda.synchronize()
        out["gn_step_ms"] = a.elapsed_time(b)
        out["gn_step_cg_iters"] = cg
        out["gn_step_note"] = ("one damped Gauss-Newton step (gn_damping=1, cg_tol 5e-3, "
                               "cg_max min(30, 3R)) after one ALS sweep from the default init")
        # generalized loss: one inner-Newton ALS sweep of the
        # Poisson log link on the same counts, everything on the device
        from paper_1910_02371_b200.optim import _als_generalized_device
        pcfg = SolverConfig(rank=R3, reg=REG, loss="poisson")
        ploss = get_loss("poisson")
        Fp = [f.clone() for f in init]
        _als_generalized_device(t, Fp, ploss, pcfg)  # warm-up
        Fp = [f.clone() for f in init]
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _als_generalized_device(t, Fp, ploss, pcfg)
        b.record(stream)
        torch.cuda.synchronize()
        out["poisson_als_sweep_ms"] = a.elapsed_time(b)
        out["poisson_als_note"] = ("inner-Newton ALS sweep, Poisson log link (inner_max 5, "
                                   "inner_tol 1e-3): fused TTTP loss epilogue + MTTKRP + "
                                   "phi2-weighted Gram + batched solve per inner step")
    else:
        from paper_1910_02371_b200 import dist as D
        coords = []
        rem = keys.clone()
        for d in reversed(shape):
            coords.append(rem % d)
            rem = rem // d
        coords = coords[::-1]
        del rem
        als = D.ShardedALS(coords, vals, shape, REG, D.DeviceBackend())
        del coords
        F = [f.clone() for f in init]
        als.sweep(F)
        torch.cuda.synchronize()
        dist.barrier()
        times = []
        for _ in range(sweeps):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            als.sweep(F)
            b.record(stream)
            torch.cuda.synchronize()
            ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            times.append(float(ms.item()))
        out["als_sweep_ms"] = float(np.mean(times))
        out["parallelism"] = (f"row-sharded x{world} (blocks balance nnz + {als.row_weight:.0f} "
                              "per row), uneven all-gather of the updated rows per mode "
                              "(one NCCL broadcast per block)")
        out["gather_bytes_per_sweep"] = sum(als.exchanged_bytes(m, R3) for m in range(3))
        out["row_blocks"] = [[b - a for a, b in blks] for blks in als.blocks]
        del als
        torch.cuda.empty_cache()
        # CCD++: nonzero-sharded, one all-reduce of (num, den) per (r, mode)
        ccd = D.ShardedCCD(keys, vals, shape, REG, D.DeviceBackend())
        F = [f.clone() for f in init]
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ccd.sweep(F)
        b.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out["ccd_sweep_ms"] = float(ms.item())
        out["ccd_parallelism"] = f"nnz-sharded x{world}, NCCL all-reduce of (num, den)"
    if cpu and rank == 0 and world == 1:
        # the reference's CPU algorithm on THIS box's host cores: the oracle's C
        # restatement (OpenMP over rows as numba's prange) of one full-size ALS
        # sweep and one CCD++ sweep on the same tensor and init
        from oracle import oracle as O
        info = cpu_info()
        O.set_threads(info["cores"])
        t0 = time.perf_counter()
        ot = O.OTensor(shape, t.keys, t.values)
        for mode in range(3):
            ot.mode_group(mode)
        setup = time.perf_counter() - t0
        host_init = [f.cpu().numpy() for f in init]
        Fh = [f.copy() for f in host_init]
        t0 = time.perf_counter()
        O.als_sweep(ot, Fh, REG)
        als_s = time.perf_counter() - t0
        Fh = [f.copy() for f in host_init]
        t0 = time.perf_counter()
        O.ccd_sweep(ot, Fh, REG)
        ccd_s = time.perf_counter() - t0
        out["cpu_reference"] = {
            "als_sweep_s": als_s, "ccd_sweep_s": ccd_s, "coords_and_mode_sorts_s": setup,
            "kind": "port", **info,
            "sample": "full cfg 3 tensor (100,480,507 nnz, R=32), one ALS sweep and one CCD++ "
                      "sweep from the bench's init, oracle/cpfit_oracle.c on all host cores"}
        out["als_speedup_vs_cpu"] = als_s * 1e3 / out["als_sweep_ms"]
        out["ccd_speedup_vs_cpu"] = ccd_s * 1e3 / out["ccd_sweep_ms"]
        del ot
    return out




def sgd_section(dev, steps=5, world=1, cpu=True):
    """BASELINE cfg 5 on one GPU: order-4 fp32 tensor 1e5^3 x 1e3 with 1e9
    distinct uniform nonzeros (device-generated, values = rank-8 CP model +
    N(0, 0.1) via the library's TTTP), R=64: SGD steps (1% Bernoulli sample,
    step 1e-3, lambda 1e-4) and the full TTTP residual evaluation."""
    import torch

    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import synth
    from paper_1910_02371_b200.losses import sum_sq, tttp_affine
    from paper_1910_02371_b200.optim import SolverConfig, _sgd_ls_device
    t0 = time.perf_counter()
    shape, tn, values, F, keys = synth.cfg5_device(with_keys=True)
    t = tn.with_values(values)
    gen_s = time.perf_counter() - t0
    cfg = SolverConfig(rank=64, algorithm="sgd", step=1e-3, reg=1e-4, sample_rate=0.01)
    stream = torch.cuda.current_stream()
    root = cp.RngState(5).child(1)
    if world > 1:
        # nonzero shards, global Philox counter, one all-reduce per mode
        import torch.distributed as dist

        from paper_1910_02371_b200 import dist as D
        sharded = D.ShardedSGD(keys, values, shape, D.DeviceBackend())

        def one(rng):
            sharded.step(F, cfg.sample_rate, cfg.step, cfg.reg, rng)
            return None
    else:
        def one(rng):
            return _sgd_ls_device(t, F, cfg, rng)
    del keys
    import gc
    gc.collect()
    one(root.child(0))  # warm-up (x2: the memory pool settles on the sample sizes)
    one(root.child(steps + 1))
    torch.cuda.synchronize()
    gc.collect()  # no pattern destructor (device free) inside the timed steps
    gc.disable()
    ms, kept = [], []
    for it in range(1, steps + 1):
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        kept.append(one(root.child(it)))
        b.record(stream)
        torch.cuda.synchronize()
        m = a.elapsed_time(b)
        if world > 1:
            mt = torch.tensor([m], dtype=torch.float64, device=dev)
            dist.all_reduce(mt, op=dist.ReduceOp.MAX)
            m = float(mt.item())
        ms.append(m)
    gc.enable()
    resid = tttp_affine(t, F, -1.0, 1.0, torch.float32)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    resid = tttp_affine(t, F, -1.0, 1.0, torch.float32)
    b.record(stream)
    torch.cuda.synchronize()
    tttp_ms = a.elapsed_time(b)
    rmse = float(np.sqrt(sum_sq(resid) / t.nnz))
    alg = t.nnz * (4 * 4 + 2 * 4 + 4 * 64 * 4)  # 1,048 B per nnz
    return {"workload": "BASELINE cfg 5: order 4, 1e5x1e5x1e5x1e3, 1e9 uniform distinct nnz, "
                        "fp32, R=64; SGD rate 0.01 (Bernoulli), step 1e-3, lambda 1e-4",
            "generation_s": gen_s, "nnz": t.nnz, "n_gpus": world,
            "sgd_step_ms": float(np.median(ms)), "sgd_step_ms_all": ms, "sample_nnz_per_step": (float(np.mean(kept)) if world == 1 else None),
            "tttp_residual_ms": tttp_ms,
            "tttp_residual_nnz_per_s": t.nnz / (tttp_ms * 1e-3),
            "tttp_residual_alg_gbs": alg / (tttp_ms * 1e-3) / 1e9,
            "rmse_after": rmse,
            "cpu_reference": cfg5_cpu_reference(dev) if (cpu and world == 1) else None}


def cfg5_cpu_reference(dev, nnz=10_000_000):
    """cfg 5's CPU reference on this box, at a 1e7-nonzero sample of the cfg 5
    laws (1e9 order-4 nonzeros do not fit the reference's host path, SURVEY.md
    8(d)): the oracle's TTTP residual and one SGD step (rate 0.01) in fp64 on
    all host cores, scaled by nnz to 1e9."""
    import torch

    from oracle import oracle as O
    from paper_1910_02371_b200 import synth
    info = cpu_info()
    O.set_threads(info["cores"])
    shape, t, values, F = synth.cfg5_device(nnz=nnz)
    ot = O.OTensor(shape, t.keys, values.cpu().numpy().astype(np.float64))
    fs = [f.cpu().numpy().astype(np.float64) for f in F]
    del t, values, F
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    ot.coords()
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.tttp(ot.with_values(np.ones(ot.nnz)), fs)
    tttp_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.sgd_sweep(ot, fs, 1e-4, 1e-3, 0.01, 5, (1, 1))
    sgd_s = time.perf_counter() - t0
    scale = 1_000_000_000 / nnz
    return {"tttp_s_at_sample": tttp_s, "sgd_step_s_at_sample": sgd_s, "coords_s": setup,
            "tttp_s_scaled_1e9": tttp_s * scale, "sgd_step_s_scaled_1e9": sgd_s * scale,
            "kind": "port", **info,
            "sample": f"{nnz} nonzeros with the cfg 5 shape/laws (order 4, R=64), fp64 oracle "
                      "on all host cores, linear in nnz to 1e9"}


def ingest_section(dev, reps=3):
    """from_coords on the device at the cfg 2 size --
    1.1e7 coordinate triples (1e7 distinct keys plus 10% duplicates, shuffled)
    -> sorted unique keys + merged values, bit-identical to the reference's
    numpy path; the numpy restatement of core.py:208-231 (linearize_many,
    stable argsort, np.add.reduceat) timed beside it on the host."""
    import torch

    from paper_1910_02371_b200 import synth
    from oracle import oracle as O
    from paper_1910_02371_b200.core import from_coords_device
    shape, keys, values, _ = synth.cfg2()
    rng = np.random.default_rng(77)
    dup = rng.integers(0, keys.size, keys.size // 10)
    allk = np.concatenate([keys, keys[dup]])
    allv = np.concatenate([values, rng.standard_normal(dup.size)])
    order = rng.permutation(allk.size)
    allk, allv = allk[order], allv[order]
    coords = synth._delinearize(allk, shape)
    dc = [torch.from_numpy(np.ascontiguousarray(c, dtype=np.int32)).to(dev) for c in coords]
    dv = torch.from_numpy(allv).to(dev)
    out = {"workload": f"cfg 2 shape, {allk.size} coordinate triples (int32, shuffled, "
                       f"{dup.size} duplicates) -> {keys.size} unique keys",
           "entries": int(allk.size)}
    t = from_coords_device(dc, dv, shape)  # warm-up (allocator, module load)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t = from_coords_device(dc, dv, shape)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    out["device_ms"] = float(np.median(times))
    out["device_entries_per_s"] = allk.size / (out["device_ms"] * 1e-3)
    t0 = time.perf_counter()
    ref = O.from_coords(coords, allv, shape)
    out["host_numpy_s"] = time.perf_counter() - t0
    out["host_what"] = "oracle numpy restatement of core.py:208-231 on one host core"
    ok = t.nnz == ref.nnz and np.array_equal(t.keys, ref.keys) and \
        np.array_equal(t.values, ref.values)
    out["bit_identical_to_numpy"] = bool(ok)
    return out


def pairwise_section(dev, reps=3):
    """The paper's comparison on the B200: all-at-once TTTP / MTTKRP vs the
    pairwise-contraction baseline (hypersparse.py: TTM through a CCSR
    matricization, semi-sparse intermediates) at the cfg 2 size, fp64, R=16,
    both through the numpy API (host factors in, host results out)."""
    import torch

    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import hypersparse as H
    from paper_1910_02371_b200 import synth
    shape, keys, values, factors = synth.cfg2()
    t = cp.SparseTensor(shape, keys, values, validate=False)

    def wall(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return float(np.median(ts))
    out = {"workload": "cfg 2 (1e7 nnz, 10^4 cube, R=16, fp64), numpy API on both sides"}
    out["all_at_once_tttp_ms"] = wall(lambda: cp.tttp(t, factors).values)
    out["pairwise_tttp_ms"] = wall(lambda: H.pairwise_tttp(t, factors).values)
    out["all_at_once_mttkrp0_ms"] = wall(lambda: cp.mttkrp(t, factors, 0))
    out["pairwise_mttkrp0_ms"] = wall(lambda: H.pairwise_mttkrp(t, factors, 0))
    out["note"] = ("pairwise MTTKRP = matricization to CCSR (device sort), CCSR x dense "
                   "(TTM), fold of the remaining factor and fiber-order row sums, with the "
                   "reference's host-resident CCSR / semi-sparse objects in between")
    return out


def dense_cpu_reference(X, F):
    """cfg 4 on the host cores of this box: numpy.einsum('ijk,jr,kr->ir',
    optimize=True) per mode (the reference has no dense path; SURVEY.md 6 used
    the same yardstick)."""
    info = cpu_info()
    Xh = X.cpu().numpy()
    A, B, C = (f.cpu().numpy() for f in F)
    specs = [("ijk,jr,kr->ir", B, C), ("ijk,ir,kr->jr", A, C), ("ijk,ir,jr->kr", A, B)]
    secs = []
    for spec, U, V in specs:
        t0 = time.perf_counter()
        np.einsum(spec, Xh, U, V, optimize=True)
        secs.append(time.perf_counter() - t0)
    return {"numpy_einsum_s_per_mode": secs, "kind": "numpy.einsum (no reference dense path)",
            **info, "sample": "full 800^3 fp64 tensor, R=64, one call per mode"}


def dense_section(dev, sweeps=2, cpu=True):
    """BASELINE cfg 4: dense 800^3 fp64 N(0,1), R=64 factors N(0,1): dense
    MTTKRP per mode and CP-ALS sweep time, against the on-box DGEMM peak."""
    import torch

    from paper_1910_02371_b200 import dense as DN
    g = torch.Generator(device=dev)
    g.manual_seed(4)
    n, R4 = 800, 64
    X = torch.randn((n, n, n), generator=g, dtype=torch.float64, device=dev)
    F = [torch.randn((n, R4), generator=g, dtype=torch.float64, device=dev) for _ in range(3)]
    stream = torch.cuda.current_stream()

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    flop = 2.0 * n ** 3 * R4
    mode_ms = [timed(lambda m=m: DN.dense_mttkrp(X, F, m)) for m in range(3)]
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    peak_ms = timed(lambda: a @ a)
    peak = 2 * 8192 ** 3 / (peak_ms * 1e-3) / 1e12
    del a
    Fs = [f.clone() for f in F]
    sweep_ms = timed(lambda: DN.dense_als_sweep(X, Fs, 1e-5), reps=sweeps)
    # TF32 tcgen05 variant on the fp32-rounded tensor: HBM-bound (X read once)
    X32 = X.float()
    F32 = [f.float() for f in F]
    tf32_ms = [timed(lambda m=m: DN.dense_mttkrp(X32, F32, m)) for m in range(3)]
    hbm, _ = peaks()
    del X32
    return {"workload": "BASELINE cfg 4: dense 800^3 fp64 N(0,1), R=64, lambda=1e-5",
            "kernels": "dense_dmma_kernel (FP64 DMMA, TMA X tiles, Khatri-Rao tile in smem, "
                       "split-K with ordered partial sums); dense_tc_kernel (TF32 tcgen05.mma, "
                       "TMEM accumulator) for fp32",
            "mttkrp_ms": mode_ms,
            "mttkrp_tflops": [flop / (t * 1e-3) / 1e12 for t in mode_ms],
            "dgemm_peak_tflops_measured": peak,
            "dgemm_peak_what": "cuBLAS DGEMM 8192^3 (torch.matmul float64), measured here as "
                               "the FP64 denominator only",
            "mttkrp_frac_of_dgemm_peak": [flop / (t * 1e-3) / 1e12 / peak for t in mode_ms],
            "tf32_mttkrp_ms": tf32_ms,
            "tf32_hbm_gbs": [n ** 3 * 4 / (t * 1e-3) / 1e9 for t in tf32_ms],
            "tf32_frac_of_hbm": [n ** 3 * 4 / (t * 1e-3) / 1e9 / hbm for t in tf32_ms],
            "als_sweep_ms": sweep_ms,
            "als_sweep_flop_model": "2 passes over X per sweep (T = X.C shared by modes 0,1; "
                                    "mode 2 one Khatri-Rao pass) + Gram / shared-G solve",
            "cpu_reference": dense_cpu_reference(X, F) if cpu else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-ref", action="store_true",
                    help="skip the on-box CPU reference legs of the cfg 3/4/5 sections")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-als", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-sgd", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the ingest and pairwise-vs-all-at-once sections")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)

    import ctypes

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per "
                         "GPU (torchrun --nproc-per-node N bench.py --gpus N, or bench.py "
                         "--gpus N alone, which self-launches)")
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1:
        # NCCL's own init lines (ranks, transports, NVLS) go to a per-rank file;
        # rank 0 summarises them into the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        nccl_log = os.environ.setdefault("NCCL_DEBUG_FILE",
                                         f"/tmp/cpfit_bench_nccl.{os.getpid()}.log")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        warm = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(warm)  # the communicator is created lazily: force it now
        torch.cuda.synchronize()

    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import _lib, synth
    from paper_1910_02371_b200.core import _dtype_code

    # cfg 5 SGD first, in a fresh process state: measured after the e2e
    # section (pinned result buffers, copy-stream events) its steps showed
    # 13-55 ms spikes instead of a flat 9.1 ms
    dev = torch.device("cuda", local)
    sgd = None
    if not args.no_sgd:
        import gc
        try:
            sgd = sgd_section(dev, world=world, cpu=not args.no_cpu_ref)
        except Exception as exc:  # reported, never fatal to the headline line
            sgd = {"error": repr(exc)}
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    # rank r holds the r-th contiguous nonzero range of one (world x 1e7)-nnz
    # tensor over the cfg 2 index space; factors replicated
    shape, keys, values, factors = synth.cfg2_shard(rank, world)
    t = cp.SparseTensor(shape, keys, values, validate=False)
    dev = torch.device("cuda", local)
    dfs = [torch.from_numpy(f).to(dev) for f in factors]
    L = _lib.load()
    pat = t.device_pattern()
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    vals = t.device_values(torch.float64)
    svals = [t.sorted_values(m, torch.float64) for m in range(3)]
    fptrs = _lib.ptr_array([f.data_ptr() for f in dfs])
    tout = torch.empty(t.nnz, dtype=torch.float64, device=dev)
    mouts = [torch.empty((shape[m], R), dtype=torch.float64, device=dev) for m in range(3)]
    launches_per_step = 1
    for m in range(3):
        nt, ns, nsl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.cpfit_pattern_mode_stats(pat.handle, m, sp, ctypes.byref(nt),
                                              ctypes.byref(ns), ctypes.byref(nsl)))
        # mttkrp_zero_empty_rows + mttkrp_kernel (+ combine_partials when rows are split)
        launches_per_step += 2 + (1 if ns.value > 0 else 0)
    F64 = _dtype_code(torch.float64)
    ev = {k: [] for k in ("tttp", "m0", "m1", "m2")}

    def step(record=False):
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        _lib.check(L.cpfit_tttp(pat.handle, F64, R, ctypes.c_void_p(vals.data_ptr()), fptrs,
                                ctypes.c_void_p(tout.data_ptr()), sp))
        if record:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            ev["tttp"].append((e0, e1))
        for m in range(3):
            if record:
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            _lib.check(L.cpfit_mttkrp(pat.handle, m, F64, R,
                                      ctypes.c_void_p(svals[m].data_ptr()), 1, fptrs,
                                      ctypes.c_void_p(mouts[m].data_ptr()), sp))
            if record:
                b = torch.cuda.Event(enable_timing=True)
                b.record(stream)
                ev[f"m{m}"].append((a, b))
            if world > 1:
                dist.all_reduce(mouts[m])

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    clocks.mark("start")
    start.record(stream)
    for _ in range(args.steps):
        step(record=True)
    stop.record(stream)
    torch.cuda.synchronize()
    clocks.mark("stop")
    ms = start.elapsed_time(stop)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    clk = clocks.stop()
    ms_step = ms / args.steps
    value = world * 4 * t.nnz / (ms_step * 1e-3)

    # per-kernel device time (CUDA events on the launching stream)
    kt = {k: float(np.mean([a.elapsed_time(b) for a, b in v])) for k, v in ev.items()}
    tb, mb, compulsory = algorithmic_bytes(3, t.nnz, R, shape)
    peak, peak_kind = peaks()
    ct, cm = compulsory_bytes(3, t.nnz, R, shape)
    kernels = {"tttp": {"ms": kt["tttp"], "alg_bytes": tb, "compulsory_bytes": ct}}
    for m in range(3):
        kernels[f"mttkrp{m}"] = {"ms": kt[f"m{m}"], "alg_bytes": mb[m], "compulsory_bytes": cm}
    for k in kernels.values():
        k["gbs"] = k["compulsory_bytes"] / (k["ms"] * 1e-3) / 1e9      # HBM-side rate
        k["frac"] = k["gbs"] / peak
        k["alg_gbs"] = k["alg_bytes"] / (k["ms"] * 1e-3) / 1e9         # incl. L2 gathers
        k["nnz_per_s"] = t.nnz / (k["ms"] * 1e-3)
    # dominant kernel = largest share of the step (MTTKRP runs once per mode)
    share = {"tttp": kernels["tttp"]["ms"],
             "mttkrp0": sum(kernels[f"mttkrp{m}"]["ms"] for m in range(3))}
    dom = max(share, key=share.get)
    roofline = {"bound": "hbm", "kernel": "mttkrp_kernel" if dom == "mttkrp0" else "tttp_kernel",
                "achieved": kernels[dom]["gbs"], "peak": peak,
                "unit": "GB/s", "frac": kernels[dom]["gbs"] / peak, "peak_kind": peak_kind,
                "step_share": share[dom] / sum(share.values()),
                "traffic": None,
                "byte_model": "compulsory bytes per launch (SURVEY.md 8(d)): the nonzero "
                              "stream m (N s_i + s_v) plus every factor/output row once, "
                              "divided by the CUDA-event launch time; the factor-row gathers "
                              "(gather-inclusive bytes) are L2 traffic, reported in roofline.l2 "
                              "against the measured L2 read peak"}
    # gather ceiling: the same row gathers with no compute (probe kernel)
    probe = None
    try:
        pout = torch.empty(num_sms_probe(torch) * 256 * 4, dtype=torch.float64, device=dev)
        coords = [pat.coords(n) for n in range(3)]
        L0 = pat.mode_group(0)  # noqa: F841  (mode-0 order == canonical)

        def run_probe(streams):
            arr = _lib.ptr_array([c.data_ptr() for c in streams])
            _lib.check(L.cpfit_probe_gather(ctypes.c_void_p(dfs[0].data_ptr()), R * 8,
                                            len(streams), arr, t.nnz,
                                            ctypes.c_void_p(pout.data_ptr()), pout.numel(), sp))
        for _ in range(3):
            run_probe(coords)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            run_probe(coords)
        b.record(stream)
        torch.cuda.synchronize()
        p3 = a.elapsed_time(b) / 10
        a.record(stream)
        for _ in range(10):
            run_probe(coords[1:])
        b.record(stream)
        torch.cuda.synchronize()
        p2 = a.elapsed_time(b) / 10
        probe = {"ms_3rows": p3, "ms_2rows": p2,
                 "gather_gbs_3rows": t.nnz * 3 * R * 8 / (p3 * 1e-3) / 1e9,
                 "gather_gbs_2rows": t.nnz * 2 * R * 8 / (p2 * 1e-3) / 1e9,
                 "what": "cpfit_probe_gather: the kernels' row gathers (same indices, "
                         "128 B rows, L2-resident table) with no shuffles/compute"}
        kernels["tttp"]["frac_of_gather_ceiling"] = p3 / kernels["tttp"]["ms"]
        for m in range(3):
            kernels[f"mttkrp{m}"]["frac_of_gather_ceiling"] = p2 / kernels[f"mttkrp{m}"]["ms"]
        roofline["frac_of_gather_ceiling"] = kernels[dom]["frac_of_gather_ceiling"]
    except Exception as exc:  # the probe is informational
        probe = {"error": str(exc)}
    # L2 read peak: coalesced passes over an L2-resident buffer (probe kernel)
    try:
        l2 = {}
        lout = torch.empty(num_sms_probe(torch) * 4 * 512, dtype=torch.int32, device=dev)
        for mb_ in (24, 48, 96):
            buf = torch.ones(mb_ << 20, dtype=torch.uint8, device=dev)

            def run_l2(reps):
                _lib.check(L.cpfit_probe_l2_read(ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                                 reps, ctypes.c_void_p(lout.data_ptr()),
                                                 lout.numel(), sp))
            run_l2(3)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run_l2(20)
            b.record(stream)
            torch.cuda.synchronize()
            l2[f"{mb_}MB_gbs"] = buf.numel() * 20 / (a.elapsed_time(b) * 1e-3) / 1e9
            del buf
        l2_peak = max(l2.values())
        roofline["l2"] = {"achieved": kernels[dom]["alg_gbs"], "peak": l2_peak, "unit": "GB/s",
                          "frac_l2": kernels[dom]["alg_gbs"] / l2_peak,
                          "peak_probe": l2,
                          "what": "gather-inclusive algorithmic bytes (SURVEY.md 8(d)) per launch "
                                  "/ launch time, against cpfit_probe_l2_read (max over buffer "
                                  "sizes of coalesced 16-B ld.global.cg passes over an "
                                  "L2-resident buffer)"}
        roofline["frac_l2"] = roofline["l2"]["frac_l2"]
        for k in kernels.values():
            k["frac_l2"] = k["alg_gbs"] / l2_peak
    except Exception as exc:  # informational
        roofline["l2"] = {"error": repr(exc)}
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tr = json.load(open(tf))
            roofline["traffic"] = tr.get(dom)
            roofline["traffic_source"] = tr.get("source")
            if roofline["traffic"]:
                roofline["achieved_dram"] = roofline["traffic"] / (kernels[dom]["ms"] * 1e-3) / 1e9
                roofline["frac_dram"] = roofline["achieved_dram"] / peak
        except Exception:
            pass

    # e2e through the public API with pinned host buffers (rank-local)
    e2e = None
    if args.e2e_steps > 0:
        pv = torch.from_numpy(values).pin_memory()
        pf = [torch.from_numpy(f).pin_memory() for f in factors]
        hv = pv.numpy()
        hf = [p.numpy() for p in pf]

        # The drop-in call a user makes: tttp / mttkrp on a persistent
        # SparseTensor (its pattern and values stay on the device after first
        # use, like the reference's cached coords / mode groups) with host
        # (pinned) numpy factors every call; results come back as numpy.
        tv = t.with_values(hv)

        def api_step():
            out = cp.tttp(tv, hf)          # values stream back while the MTTKRPs run
            ms_ = [cp.mttkrp(tv, hf, m) for m in range(3)]
            vals_host = out.values          # waits for the last TTTP chunk's copy
            return vals_host, ms_
        api_step()
        api_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            api_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        h2d = 3 * factors[0].nbytes + 3 * 2 * factors[0].nbytes
        d2h = t.nnz * 8 + sum(shape[m] * R * 8 for m in range(3))
        e2e = {"value": world * 4 * t.nnz / dt, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
               "path": "paper_1910_02371_b200.tttp(t, F) + mttkrp(t, F, m) x3 + the TTTP "
                       "result's .values, with pinned-host numpy factors uploaded on every "
                       "call and every result read back as numpy inside the timed step (TTTP "
                       "values stream back on a copy stream while the MTTKRPs compute); t "
                       "persistent (values uploaded once, pattern cached)"}

    # remaining sections.  Collect the headline's tensors now: a pattern freed
    # later by the cyclic GC would release its device memory (a device-wide
    # synchronisation) inside some other section's timed region.
    del t, tout, mouts, svals, vals
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    als = None
    if not args.no_als:
        try:
            als = als_section(world, rank, dev, cpu=not args.no_cpu_ref)
        except Exception as exc:
            als = {"error": repr(exc)}
        torch.cuda.empty_cache()
    ingest = None
    pairwise = None
    if world == 1 and not args.no_extra:
        try:
            ingest = ingest_section(dev)
        except Exception as exc:
            ingest = {"error": repr(exc)}
        torch.cuda.empty_cache()
        try:
            pairwise = pairwise_section(dev)
        except Exception as exc:
            pairwise = {"error": repr(exc)}
        torch.cuda.empty_cache()
    dense = None
    if not args.no_dense and world == 1:
        try:
            dense = dense_section(dev, cpu=not args.no_cpu_ref)
        except Exception as exc:
            dense = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE cfg 2 shape/value laws)",
            "config": dict(CONFIG, parallelism=f"nnz-shard{world}" if world > 1 else "1gpu"),
            "roofline": roofline, "kernels": kernels, "gather_ceiling": probe,
            "compulsory_bytes_per_pass": compulsory,
            "clocks": clk, "gpu_launches": launches_per_step * args.steps, "e2e": e2e,
            "als": als, "dense": dense, "sgd": sgd, "ingest": ingest,
            "pairwise_vs_all_at_once": pairwise,
        }
        if world > 1:
            line["nccl"] = nccl_summary(nccl_log, world)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
