#!/usr/bin/env python
"""bench.py — throughput of the reversible-AD gradient kernels on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload all|bessel|ba|gmm|gmm_large] [--dry-run]

Default (--workload all): the headline is BASELINE.json configs[1], the
Bessel J_2 gradient over a batch of 2^26 inputs z ~ U(0.1, 10) (seed 1),
sharded over the ranks (strong scaling: the 2^26 batch is fixed, each rank
takes a contiguous slice; no collective on the data path).  A "step" = one
fused forward + reverse-sweep kernel over the rank's slice, inputs resident
in HBM (512 MiB > 126 MB L2, so no flush is needed between steps).  The same
line carries one sub-object per other BASELINE config, each with its own
value, roofline, cpu_baseline, e2e and clocks: "ba" (configs[3], ba20
Jacobian), "gmm_c3" (configs[2], d=64 K=25 N=10^4) and "gmm_c5" (configs[4],
d=128 K=200 N=10^6); each is timed over >= 200 ms of device time so the
clock sampler sees it.

--gpus N > 1 without torchrun: bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL); under torchrun the
world size must equal --gpus.

Printed (rank 0, one JSON line): value = whole-job gradient evals/s from
the device time (CUDA events, max over ranks); e2e = the same metric
through the C-ABI host-buffer entry (pinned host inputs in, outputs out,
copies inside the timed region); roofline of the dominant kernel against
the in-run measured FP64 DFMA / DMMA peak (HBM for BA); cpu_baseline = the C
oracle port (oracle/, the reference algorithm) on a bounded sample; clocks
sampled with NVML during the timed region.

`--impl reference` times the reference algorithm's CPU implementation
(the oracle port — the reference itself is pure Python and cannot travel
to the GPU box) on the same workloads and configs, rank 0 only, each rate
from a bounded sample ("rate_sample": true).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

THR = 1e-16


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-graph", action="store_true",
                    help="GMM: launch the step's kernels directly instead of as a CUDA graph")
    ap.add_argument("--workload", choices=["all", "bessel", "ba", "gmm", "gmm_large"],
                    default="all")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU work: exercise the launch / world-size / max-over-ranks "
                         "plumbing under gloo (CPU tests)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: functional check of the N>1 path with every rank "
                         "folded onto the visible GPU(s) (timings meaningless)")
    ap.add_argument("--n", type=int, default=None, help="override the batch size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# environment / distributed plumbing
# ---------------------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Dist:
    def __init__(self, backend):
        import torch
        import torch.distributed as dist
        self.rank, self.world, self.local = dist_env()
        self.dist = dist if self.world > 1 else None
        self.torch = torch
        self.backend = backend
        self.nccl_log = None
        # this rank's GPU: LOCAL_RANK on an N-GPU node; folded onto the visible
        # devices only for the single-GPU functional check (--dist-backend gloo)
        self.gpu = self.local
        if torch.cuda.is_available() and backend != "nccl":
            self.gpu = self.local % torch.cuda.device_count()
        if self.dist is not None:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl" and torch.cuda.is_available():
                # the communicator's own INIT lines (nRanks, NVLS/P2P) to a
                # per-rank file, summarised into the JSON line
                self.nccl_log = f"/tmp/bench_nccl.{os.getpid()}.log"
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", self.nccl_log)
                # bind this rank to its GPU before the communicator is created
                torch.cuda.set_device(self.gpu)
                dist.init_process_group(backend, device_id=torch.device("cuda", self.gpu))
            else:
                if torch.cuda.is_available():
                    torch.cuda.set_device(self.gpu)
                dist.init_process_group(backend)
            if dist.get_world_size() != self.world:
                raise SystemExit(f"world size {dist.get_world_size()} != WORLD_SIZE {self.world}")

    def nccl_info(self):
        """nRanks / version lines of this rank's communicator (NCCL_DEBUG=INFO)."""
        if self.dist is None:
            return None
        info = {"backend": self.backend, "world_size": self.dist.get_world_size()}
        path = os.environ.get("NCCL_DEBUG_FILE")
        if path and os.path.exists(path):
            with open(path, errors="replace") as fh:
                txt = fh.read()
            import re
            m = re.findall(r"nRanks (\d+)", txt)
            if m:
                info["nccl_nranks"] = int(m[-1])
            v = re.search(r"NCCL version ([\w.+-]+)", txt)
            if v:
                info["nccl_version"] = v.group(1)
            info["nvls"] = "NVLS" in txt and "NVLS multicast support is not available" not in txt
        return info

    def _dev(self):
        return "cuda" if self.backend == "nccl" and self.torch.cuda.is_available() else "cpu"

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x):
        if self.dist is None:
            return x
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if self.dist is None:
            return x
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self._dev())
        self.dist.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    (pynvml, every ~2 ms in a thread, so even a few-ms region gets samples),
    with nvidia-smi -lms 200 as the fallback when NVML is unavailable."""

    QUERY = ("index,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, uuid=None):
        self.uuid = uuid
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []
        self.stop_evt = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        if self.uuid:
            try:
                return pynvml, pynvml.nvmlDeviceGetHandleByUUID(self.uuid)
            except pynvml.NVMLError:
                pass
        idx = int((os.environ.get("CUDA_VISIBLE_DEVICES") or "0").split(",")[0] or 0) \
            if (os.environ.get("CUDA_VISIBLE_DEVICES") or "0").split(",")[0].isdigit() else 0
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def start(self):
        try:
            self.nv = self._nvml_handle()
        except Exception:  # noqa: BLE001 - NVML missing: fall back to nvidia-smi
            self.nv = None
        if self.nv is not None:
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        cmd = ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
               "-lms", "200"]
        if self.uuid:
            cmd[1:1] = ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.25)                   # nvidia-smi needs a moment for its first line

    def _poll(self):
        nv, h = self.nv
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop_evt.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, smax, {k for k, b in bits.items() if r & b}))
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.stop_evt.set()
            self.thread.join(timeout=2)
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            reasons = set().union(*(x[2] for x in self.samples))
            return {"sm_mhz": statistics.median(x[0] for x in self.samples),
                    "sm_max_mhz": max(x[1] for x in self.samples), "reasons": sorted(reasons),
                    "samples": len(self.samples), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 10:
                continue
            try:
                sm.append(float(parts[2]))
                smax.append(float(parts[3]))
            except ValueError:
                continue
            for nm, flag in zip(self.NAMES, parts[6:10]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def time_device(fn, steps, flush=None):
    """Mean device ms of fn() over `steps` launches (CUDA events on the current
    stream; optional L2 flush between launches, outside the events)."""
    import torch
    stream = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


def load_weights():
    p = os.path.join(REPO, "profiles", "fp64_weights.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return None


def fp64_peak_tflops():
    """In-run DFMA-bound microkernel (tools/fp64probe.cu): MEASURED_PEAKS.json
    carries no FP64 figure and B200_PROFILING.md states no FP64 fallback."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(REPO, "tools", "libfp64probe.so"))
    lib.probe_dfma_peak.restype = ctypes.c_double
    lib.probe_dfma_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    ms = ctypes.c_float(0)
    best = 0.0
    for _ in range(3):
        best = max(best, lib.probe_dfma_peak(20000, ctypes.byref(ms)))
    return best, float(ms.value)


def dmma_peak_tflops():
    """In-run FP64 tensor-core (DMMA mma.sync.m16n8k16.f64) microkernel: the
    peak of the unit GMM's tile products run on (tools/fp64probe.cu)."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(REPO, "tools", "libfp64probe.so"))
    lib.probe_dmma_peak.restype = ctypes.c_double
    lib.probe_dmma_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    ms = ctypes.c_float(0)
    return max(lib.probe_dmma_peak(1, 2000, ctypes.byref(ms)) for _ in range(3))


# ---------------------------------------------------------------------------
# Bessel workload (configs[1])
# ---------------------------------------------------------------------------

BESSEL_N = 1 << 26
BESSEL_NU = 2


def bessel_config(n_total, world):
    return {"workload": "bessel_j2_grad_2^26" if n_total == BESSEL_N else f"bessel_j2_grad_{n_total}",
            "n_total": n_total, "nu": BESSEL_NU, "thr": THR, "per_rank": n_total // world,
            "parallelism": f"shard{world}", "l2": "inputs 512 MiB > 126 MB L2; no flush"}


def bessel_flops(n, sum_trips, nu, w):
    """Algorithmic FP64 flops of one launch (DESIGN.md §Bessel roofline):
    per series trip  forward 3 add + exp + 1 add; reverse 1 add + 1 mul +
    1 add + 3 add + 1 add + exp  -> 11 + 2 w_exp;
    per element      log(z) + 5 + 2 nu + exp  (prologue) and
                     12 + 3 nu + div (epilogue)."""
    per_trip = 11 + 2 * w["exp"]
    per_elem = w["log"] + w["exp"] + w["div"] + 17 + 5 * nu
    return sum_trips * per_trip + n * per_elem


def bessel_inputs(torch, n_total, rank, world, device):
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    g = torch.Generator(device=device)
    g.manual_seed(1)
    z = torch.empty(n_total, dtype=torch.float64, device=device)
    z.uniform_(0.1, 10.0, generator=g)
    return z[lo:hi].contiguous(), lo, hi


def run_bessel_ours(args, D):
    import torch

    import paper_2003_04617_b200 as rg
    from paper_2003_04617_b200 import kernels

    dev = torch.device("cuda", D.gpu)
    torch.cuda.set_device(dev)
    n_total = args.n or BESSEL_N
    z, lo, hi = bessel_inputs(torch, n_total, D.rank, D.world, dev)
    n = z.numel()
    J = torch.empty_like(z)
    dz = torch.empty_like(z)
    fail = torch.empty(n, dtype=torch.uint8, device=dev)
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    out = (J, dz, fail)
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 3)):
        kernels.besselj_grad(z, BESSEL_NU, out=out, counters=counters)
    torch.cuda.synchronize()
    counters.zero_()
    props = torch.cuda.get_device_properties(dev)
    sampler = ClockSampler(getattr(props, "uuid", None) and f"GPU-{props.uuid}")
    sampler.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        kernels.besselj_grad(z, BESSEL_NU, out=out, counters=counters)
    ev1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    ms_step = D.max(ms_total / args.steps)
    sum_trips = int(counters[0].item()) // args.steps
    n_failed = int(counters[1].item()) // args.steps
    value = n_total / (ms_step * 1e-3)

    # parity spot check of this run's outputs against the oracle (rank 0 sample)
    parity = None
    if D.rank == 0:
        parity = bessel_spot_parity(z, J, dz, fail)

    # roofline of k_besselj_grad (the only kernel of the step)
    w = load_weights()
    peak, peak_ms = fp64_peak_tflops()
    roof = None
    if w is not None:
        fl = D.sum(bessel_flops(n, sum_trips, BESSEL_NU, w))
        achieved = fl / (ms_step * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                "peak_source": "in-run DFMA microkernel (tools/fp64probe.cu); no FP64 "
                               "figure in MEASURED_PEAKS.json or B200_PROFILING.md",
                "flops_per_launch": fl, "weights": w.get("source", "profiles/fp64_weights.json")}
        tr = load_traffic("k_besselj<1>")
        if tr:
            roof["traffic"] = tr
        # cross-check: FP64 flops ncu counted for one configs[1] launch (2 per
        # DFMA, 1 per DADD / DMUL; profiles/r01/ncu_bessel_flops.json) over
        # this run's device time
        fp = os.path.join(REPO, "profiles", "r01", "ncu_bessel_flops.json")
        if os.path.exists(fp) and n_total == 1 << 26:
            with open(fp) as fh:
                ex = json.load(fh)["executed_fp64_flops"]
            roof["executed_flops_per_launch_ncu"] = ex
            roof["executed_frac"] = round(ex / (ms_step * 1e-3) / 1e12 / peak, 4)
    # objective only ("-O", the paper's objective timing): run of besselj
    o_ms = D.max(time_device(lambda: kernels.besselj_run(z, BESSEL_NU), max(3, args.steps // 4)))
    objective = {"ms_per_step": round(o_ms, 4), "grad_over_objective": round(ms_step / o_ms, 3),
                 "kernel": "k_besselj<0> (rl_besselj_run_f64)"}
    # forward-over-reverse Hessian (d2J/dz2 with J and dJ/dz) of the same batch
    h_ms = D.max(time_device(lambda: kernels.besselj_hess(z, BESSEL_NU), max(3, args.steps // 4)))
    # the same gradient through the generic .rnl -> CUDA compiler (codegen.py)
    generic = None
    try:
        from paper_2003_04617_b200 import codegen
        ck = codegen.compile_function(open(os.path.join(REPO, "paper_2003_04617_b200", "programs",
                                                        "besselj.rnl")).read(),
                                      "besselj", int_params=("nu",))
        g_ms = D.max(time_device(lambda: ck.gradient({"out!": 0.0, "z": z, "nu": BESSEL_NU}),
                                 max(2, args.steps // 8)))
        generic = {"ms_per_step": round(g_ms, 4), "over_handwritten": round(g_ms / ms_step, 2),
                   "kernel": "codegen.compile_function(programs/besselj.rnl)"}
    except Exception as err:  # noqa: BLE001 - reported, not fatal to the bench line
        generic = {"unavailable": str(err)[:200]}
    hess = {"ms_per_step": round(h_ms, 4), "hessians_per_s": round(n_total / (h_ms * 1e-3), 1),
            "hess_over_grad": round(h_ms / ms_step, 3),
            "kernel": "k_besselj<2> (rl_besselj_hess_f64, Dual-number sweeps)"}
    e2e = None
    if not args.no_e2e:
        e2e = bessel_e2e(torch, z, args, D, n_total)
    res = {
        "metric": "gradient evals/sec", "value": round(value, 1), "unit": "grads/s",
        "n_gpus": D.world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic z ~ U(0.1, 10), seed 1",
        "config": bessel_config(n_total, D.world),
        "roofline": roof, "e2e": e2e, "gpu_launches": args.steps,
        "clocks": clocks, "sum_trips_per_step": D.sum(sum_trips),
        "failed_per_step": D.sum(n_failed), "parity_sample": parity,
        "objective_only": objective, "hessian": hess, "generic_codegen": generic,
    }
    return res


def bessel_spot_parity(z, J, dz, fail, m=4096):
    """The GPU outputs of the timed run vs the oracle on a strided sample."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    idx = np.linspace(0, z.numel() - 1, m).astype(np.int64)
    zs = z.cpu().numpy()[idx]
    Jo, dzo, fo, _ = O.besselj_grad(BESSEL_NU, zs)
    Jg, dzg = J.cpu().numpy()[idx], dz.cpu().numpy()[idx]
    fg = fail.cpu().numpy()[idx]
    err = lambda a, b: float(np.max(np.abs(a - b) / (np.abs(b) + 1e-2)))  # noqa: E731
    return {"n": m, "max_rel_J": err(Jg, Jo), "max_rel_dJdz": err(dzg, dzo),
            "flags_equal": bool(np.array_equal(fg, fo))}


def bessel_e2e(torch, z, args, D, n_total):
    """Host buffers through the C-ABI `_host` entry: H2D + kernels + D2H."""
    from paper_2003_04617_b200 import kernels
    n = z.numel()
    zh = z.cpu().pin_memory()
    Jh = torch.empty(n, dtype=torch.float64).pin_memory()
    dzh = torch.empty(n, dtype=torch.float64).pin_memory()
    fh = torch.empty(n, dtype=torch.uint8).pin_memory()
    outs = (Jh.numpy(), dzh.numpy(), fh.numpy())
    zn = zh.numpy()
    steps = max(2, min(args.steps, 5))
    kernels.besselj_grad_host(zn, BESSEL_NU, out=outs, device=D.gpu)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        kernels.besselj_grad_host(zn, BESSEL_NU, out=outs, device=D.gpu)
    dt = D.max((time.perf_counter() - t0) / steps)
    # per rank: z up; J and dJ/dz down, plus per 4 Mi-element chunk a count
    # and a 16384-entry list of the nonzero status codes (capi.cu)
    nch = -(-n // (1 << 22))
    d2h = D.sum(16 * n + nch * (16384 * 4 + 4))
    return {"value": round(n_total / dt, 1), "unit": "grads/s", "h2d_bytes_per_step": 8 * n_total,
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 3),
            "path": "rl_besselj_grad_f64_host (pinned host buffers, 3-stream pipeline; status "
                    "codes as per-chunk lists of the failures)"}


def bessel_cpu(target_s=2.0, n_max=1 << 24):
    """The oracle port over all host threads on a bounded sample."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    rng = np.random.default_rng(1)
    cores = os.cpu_count() or 1
    n = 4096
    while True:
        z = rng.uniform(0.1, 10.0, n)
        t0 = time.perf_counter()
        O.besselj_grad(BESSEL_NU, z)
        dt = time.perf_counter() - t0
        if dt >= target_s or n >= n_max:
            break
        n = min(n_max, max(n * 2, int(n * target_s / max(dt, 1e-3))))
    threads = int(os.environ.get("OMP_NUM_THREADS", cores))
    return {"value": round(n / dt, 1), "unit": "grads/s", "cores": threads, "kind": "port",
            "sample": f"{n} z ~ U(0.1,10) of the 2^26 workload, all 4 reference sweeps with "
                      f"checks (oracle/revoracle.c), {dt:.2f} s"}


def gmm_traffic():
    """DRAM bytes of one configs[2] GMM evaluation: the round-2 measurement
    with L2 evicted before the evaluation and no flush between its kernels
    (profiles/r02/gmm_c3_dram_per_eval.json, tools/gmm_one.py --flush under
    ncu --cache-control none), else the per-kernel cold-cache sum."""
    p2 = os.path.join(REPO, "profiles", "r02", "gmm_c3_dram_per_eval.json")
    if os.path.exists(p2):
        with open(p2) as fh:
            return int(json.load(fh)["total_MB"] * 1e6)
    p = os.path.join(REPO, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    v = [b for k, b in d.items() if k.startswith("k_gmm")]
    return int(sum(v)) if v else None


def load_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture at the
    bench's problem size (profiles/traffic.json, tools/make_traffic.py)."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        for k, v in d.items():
            if not k.startswith("_") and (k == kernel or k.startswith(kernel + "<")
                                          or k.replace("rl::", "") == kernel):
                return v
    return None


# ---------------------------------------------------------------------------
# BA workload (configs[3], ba20 shape)
# ---------------------------------------------------------------------------

BA_N, BA_M, BA_P = 1723, 156502, 678718


def ba_synthetic(n_cams, n_pts, n_obs, seed=3):
    rng = np.random.default_rng(seed)
    cams = np.empty((n_cams, 11))
    cams[:, 0:3] = rng.normal(0.0, 0.3, (n_cams, 3))
    cams[:, 3:6] = rng.normal(0.0, 1.0, (n_cams, 3))
    cams[:, 6] = rng.uniform(500.0, 600.0, n_cams)
    cams[:, 7:9] = rng.uniform(0.0, 1.0, (n_cams, 2))
    cams[:, 9:11] = rng.normal(0.0, 0.01, (n_cams, 2))
    X = rng.normal(0.0, 1.0, (n_pts, 3))
    X[:, 2] += 10.0
    w = rng.uniform(0.0, 1.0, n_obs)
    feats = rng.uniform(0.0, 100.0, (n_obs, 2))
    i = np.arange(n_obs)
    obs = np.stack([i % n_cams, i % n_pts], 1).astype(np.int32)
    return cams, X, w, feats, obs


def ba_config(p_total, world):
    return {"workload": "ba20_jacobian", "n_cams": BA_N, "n_pts": BA_M, "n_obs": p_total,
            "per_rank": p_total // world, "parallelism": f"shard{world}",
            "l2": "256 MiB L2 flush before every timed launch; per-launch CUDA events"}


def steps_for(step_ms, args, floor_ms=200.0, budget_ms=2000.0, cap=20000):
    """Timed steps of a sub-workload: at least 3 and at least floor_ms of
    device time (so the NVML clock sampler sees the region), and --steps when
    that fits in budget_ms."""
    step_ms = max(step_ms, 1e-3)
    n = max(3, -(-floor_ms // step_ms))
    n = max(n, min(args.steps, budget_ms // step_ms))
    return int(min(cap, n))


def ba_bytes(n_cams, n_pts, p):
    """Algorithmic HBM bytes of one Jacobian launch (DESIGN.md §BA roofline):
    read obs (8) + w (8) + feats (16) per observation, every camera (88) and
    point (24) once; write the 31-double Jacobian row (248)."""
    return p * (8 + 8 + 16 + 248) + n_cams * 88 + n_pts * 24


def run_ba_ours(args, D):
    import torch

    from paper_2003_04617_b200 import kernels
    dev = torch.device("cuda", D.gpu)
    torch.cuda.set_device(dev)
    p_total = args.n or BA_P
    cams, X, w, feats, obs = ba_synthetic(BA_N, BA_M, p_total)
    lo, hi = p_total * D.rank // D.world, p_total * (D.rank + 1) // D.world
    t = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    dc, dX, dw, df, do = t(cams), t(X), t(w[lo:hi]), t(feats[lo:hi]), t(obs[lo:hi])
    p = hi - lo
    J = torch.empty((p, 31), dtype=torch.float64, device=dev)
    fail = torch.empty(p, dtype=torch.uint8, device=dev)
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = (J, None, None, fail)
    for _ in range(max(args.warmup, 3)):
        kernels.ba_jacobian(dc, dX, dw, df, do, want_err=False, out=out, counters=counters)
    torch.cuda.synchronize()
    props = torch.cuda.get_device_properties(dev)
    stream = torch.cuda.current_stream()
    steps = steps_for(D.max(time_device(
        lambda: kernels.ba_jacobian(dc, dX, dw, df, do, want_err=False, out=out),
        3, flush) + 0.05), args)
    counters.zero_()
    sampler = ClockSampler(getattr(props, "uuid", None) and f"GPU-{props.uuid}")
    sampler.start()
    D.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        flush.fill_(1)                      # evict L2 (inputs are 26 MB < 126 MB L2)
        a.record(stream)
        kernels.ba_jacobian(dc, dX, dw, df, do, want_err=False, out=out, counters=counters)
        b.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    ms_step = D.max(ms)
    n_failed = D.sum(int(counters[1].item()))
    value = 1.0 / (ms_step * 1e-3)
    byts = ba_bytes(BA_N, BA_M, p)
    achieved = D.sum(byts) / (ms_step * 1e-3) / 1e9
    peak = measured_hbm()
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": load_traffic("k_ba_jac"),
            "bytes_per_launch": D.sum(byts), "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    parity = None
    if D.rank == 0:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle as O
        idx = np.linspace(0, p - 1, 2000).astype(np.int64)
        Jo, _, fo = O.ba_jac(cams, X, w[lo:hi][idx], feats[lo:hi][idx], obs[lo:hi][idx])
        Jg = J.cpu().numpy()[idx]
        sc = np.max(np.abs(Jo), axis=1, keepdims=True)
        parity = {"n": 2000, "max_err_over_rowscale": float(np.max(np.abs(Jg - Jo) / sc)),
                  "flags_equal": bool(np.array_equal(fail.cpu().numpy()[idx], fo))}
    o_ms = D.max(time_device(lambda: kernels.ba_residuals(dc, dX, dw, df, do),
                             max(3, args.steps // 4), flush))
    objective = {"ms_per_step": round(o_ms, 4), "grad_over_objective": round(ms_step / o_ms, 3),
                 "kernel": "k_ba_jac<true,false,false> (rl_ba_residuals_f64)"}
    # the same Jacobian as ADBench's BASparseMat (CSR values + int32 pattern)
    csr_out = (torch.empty(3 * p + 1, dtype=torch.int32, device=dev),
               torch.empty(31 * p, dtype=torch.int32, device=dev),
               torch.empty(31 * p, dtype=torch.float64, device=dev), fail, None)
    c_ms = D.max(time_device(lambda: kernels.ba_jacobian_csr(
        dc, dX, dw, df, do, obs_offset=lo, n_obs_total=p_total, out=csr_out, counters=counters),
        max(3, args.steps // 4), flush))
    c_bytes = byts + p * (31 * 4 + 3 * 4) + 4
    csr = {"ms_per_step": round(c_ms, 4), "kernel": "k_ba_jac<..,CSR> (rl_ba_jac_csr_f64)",
           "bytes_per_launch": D.sum(c_bytes),
           "achieved_gbs": round(D.sum(c_bytes) / (c_ms * 1e-3) / 1e9, 1),
           "frac": round(D.sum(c_bytes) / (c_ms * 1e-3) / 1e9 / peak, 4)}
    # SURVEY §8(d)'s gather-stress variant: the same observations with the
    # point indices shuffled (camera rows still i mod n), so consecutive
    # observations gather scattered points
    obs_sh = obs[lo:hi].copy()
    obs_sh[:, 1] = np.random.default_rng(33).permutation(obs_sh[:, 1])
    dsh = t(obs_sh)
    s_ms = D.max(time_device(lambda: kernels.ba_jacobian(dc, dX, dw, df, dsh, want_err=False,
                                                         out=out),
                             max(3, args.steps // 4), flush))
    shuffled = {"ms_per_step": round(s_ms, 4), "value": round(1.0 / (s_ms * 1e-3), 2),
                "frac": round(D.sum(byts) / (s_ms * 1e-3) / 1e9 / peak, 4),
                "obs": "point index permuted (seed 33), camera index i mod n"}
    e2e = None
    if not args.no_e2e:
        e2e = ba_e2e(cams, X, w[lo:hi], feats[lo:hi], obs[lo:hi], args, D)
    return {
        "metric": "Jacobian evals/sec", "value": round(value, 2), "unit": "jacobians/s",
        "n_gpus": D.world, "steps": steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic ba20-shaped problem, seed 3",
        "config": ba_config(p_total, D.world),
        "obs_per_s": round(p_total / (ms_step * 1e-3), 1),
        "roofline": roof, "e2e": e2e, "gpu_launches": steps, "clocks": clocks,
        "failed_per_step": n_failed // steps, "parity_sample": parity,
        "objective_only": objective, "csr_jacobian": csr, "shuffled_obs": shuffled,
    }


def ba_e2e(cams, X, w, feats, obs, args, D):
    import ctypes

    import torch

    from paper_2003_04617_b200 import _native
    L = _native.lib()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hc, hX, hw, hf, ho = pin(cams), pin(X), pin(w), pin(feats), pin(obs)
    p = w.size
    hJ = torch.empty((p, 31), dtype=torch.float64).pin_memory()
    hfl = torch.empty(p, dtype=torch.uint8).pin_memory()
    nf = ctypes.c_ulonglong()

    def call():
        rc = L.rl_ba_jac_f64_host(cams.shape[0], X.shape[0], p, hc.data_ptr(), hX.data_ptr(),
                                  hw.data_ptr(), hf.data_ptr(), ho.data_ptr(), 1e-9, 1, None,
                                  hJ.data_ptr(), hfl.data_ptr(), ctypes.byref(nf), D.gpu)
        _native.check(rc, "rl_ba_jac_f64_host")
    call()
    D.barrier()
    steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = D.max((time.perf_counter() - t0) / steps)
    h2d = cams.nbytes + X.nbytes + D.sum(w.nbytes + feats.nbytes + obs.nbytes)
    return {"value": round(1.0 / dt, 2), "unit": "jacobians/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(D.sum(hJ.numel() * 8 + p)),
            "ms_per_step": round(dt * 1e3, 3),
            "path": "rl_ba_jac_f64_host (pinned host buffers, 3-stream pipeline)"}


def ba_cpu(target_s=2.0):
    """Whole Jacobians (all observations) repeated until ~target_s of wall time
    over all host threads."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    cams, X, w, feats, obs = ba_synthetic(BA_N, BA_M, BA_P)
    reps = 0
    t0 = time.perf_counter()
    while True:
        O.ba_jac(cams, X, w, feats, obs)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= target_s:
            break
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": round(reps / dt, 4), "unit": "jacobians/s", "cores": cores, "kind": "port",
            "obs_per_s": round(reps * BA_P / dt, 1),
            "sample": f"{reps} full Jacobians ({BA_P} observations each: 2 seeded passes + "
                      f"weight, all reference sweeps and checks, oracle/revoracle.c), {dt:.2f} s"}


def measured_hbm():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"])
    return 6650.0  # B200_PROFILING.md fallback


# ---------------------------------------------------------------------------
# GMM workloads (configs[2] d=64 K=25 N=1e4; configs[4] d=128 K=200 N=1e6)
# ---------------------------------------------------------------------------

GMM_CFG = {"gmm": (64, 25, 10000, 2), "gmm_large": (128, 200, 1000000, 4)}


def gmm_constants(d, K, N, gamma, m):
    import math
    n = d + m + 1
    lgd = 0.25 * d * (d - 1) * math.log(math.pi) + sum(
        math.lgamma(0.5 * n + 0.5 * (1 - j)) for j in range(1, d + 1))
    C = n * d * (math.log(gamma) - 0.5 * math.log(2.0)) - lgd
    return -N * d * 0.5 * math.log(2.0 * math.pi) - K * C


def gmm_flops(d, K, N, w):
    """W = 4 N K (d^2 + 3d + 3) + N K (2 w_exp + 8) + 2 N w_log
    (forward + reverse recompute + 2 adjoint mat-vec passes per point and
    component, plus the logsumexp)."""
    return 4.0 * N * K * (d * d + 3 * d + 3) + N * K * (2 * w["exp_libdevice"] + 8) + \
        2.0 * N * w["log"]


def gmm_data(seed):
    return (f"synthetic SURVEY §8(d): alphas~N(0,1), means~U(0,1), icf~N(0,1), x~U(0,1), "
            f"gamma=1, m=0, seed {seed}")


def gmm_config(d, K, N, world):
    return {"workload": f"gmm_d{d}_K{K}_N{N}", "d": d, "K": K, "N": N,
            "per_rank": N // world,
            "parallelism": "dp1" if world == 1 else f"dp{world}+allreduce",
            "l2": "256 MiB L2 flush before every evaluation"}


def gmm_inputs(torch, d, K, N, seed, lo, hi, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    alphas = torch.randn(K, dtype=torch.float64, device=dev, generator=g)
    means = torch.rand((K, d), dtype=torch.float64, device=dev, generator=g)
    icf = torch.randn((K, d * (d + 1) // 2), dtype=torch.float64, device=dev, generator=g)
    x = torch.empty((hi - lo, d), dtype=torch.float64, device=dev)
    # the rank's slice of one global x ~ U(0,1) (generated in 1M-row pieces)
    gx = torch.Generator(device=dev)
    gx.manual_seed(seed + 1)
    row = 0
    while row < hi:
        n = min(1 << 20, N - row)
        blk = torch.rand((n, d), dtype=torch.float64, device=dev, generator=gx)
        a, b = max(row, lo), min(row + n, hi)
        if a < b:
            x[a - lo:b - lo] = blk[a - row:b - row]
        row += n
    return alphas, means, icf, x


def run_gmm_ours(args, D, wl):
    """One GMM config.  One GPU: the drop-in gradient() of the whole problem
    (rl_gmm_gradient_f64: err! in the program's order and the primal-
    restoration verdict, k_gmm_restore beside k_gmm_rev).  N GPUs: each rank
    the shard entry over its points (rl_gmm_grad_f64), then ONE NCCL
    all_reduce(sum) of the packed [err, g_alphas, g_means, g_icf] vector."""
    import torch

    from paper_2003_04617_b200 import _native, kernels
    dev = torch.device("cuda", D.gpu)
    torch.cuda.set_device(dev)
    d, K, N, seed = GMM_CFG[wl]
    N = args.n if (args.n and args.workload == wl) else N
    gamma, m = 1.0, 0
    cst = gmm_constants(d, K, N, gamma, m)
    lo, hi = N * D.rank // D.world, N * (D.rank + 1) // D.world
    alphas, means, icf, x = gmm_inputs(torch, d, K, N, seed, lo, hi, dev)
    L = _native.lib()
    ws = torch.empty(max(1, L.rl_gmm_workspace_bytes(d, K, hi - lo)), dtype=torch.uint8, device=dev)
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    single = D.dist is None

    def step():
        if single:
            return kernels.gmm_gradient(alphas, means, icf, x, gamma, m, cst, workspace=ws,
                                        counters=counters)
        r = kernels.gmm_grad(alphas, means, icf, x, gamma, m, cst, N_total=N,
                             add_param_terms=(D.rank == 0), workspace=ws, counters=counters)
        D.dist.all_reduce(r.packed)            # the one collective: parameter adjoints
        return r

    for _ in range(max(args.warmup, 3)):
        r = step()
    torch.cuda.synchronize()
    # the step's launches (prep, fwd, lse, rev || restore, final) are replayed
    # as one CUDA graph: no per-launch host latency between them
    graph = None
    if not args.no_graph and single:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            r = step()
        graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    steps = steps_for(D.max(time_device(run_step, 2, flush)), args)
    counters.zero_()
    props = torch.cuda.get_device_properties(dev)
    sampler = ClockSampler(getattr(props, "uuid", None) and f"GPU-{props.uuid}")
    sampler.start()
    stream = torch.cuda.current_stream()
    D.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        flush.fill_(1)                      # evict L2 between evaluations
        a.record(stream)
        run_step()
        b.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    ms_step = D.max(ms)
    n_failed = D.sum(int(counters[1].item())) // steps
    w = load_weights()
    # GMM's mat-vec work runs on the FP64 tensor cores: the roofline peak is
    # the larger of the measured DMMA and DFMA peaks (the DMMA one)
    dfma, _ = fp64_peak_tflops()
    dmma = dmma_peak_tflops()
    peak = max(dfma, dmma)
    roof = None
    if w is not None:
        fl = gmm_flops(d, K, N, w)
        P = d * (d + 1) // 2
        executed = 2.0 * 3 * N * K * P
        roof = {"bound": "fp64", "achieved": round(fl / (ms_step * 1e-3) / 1e12, 3),
                "peak": round(peak, 3), "unit": "TFLOP/s",
                "frac": round(fl / (ms_step * 1e-3) / 1e12 / peak, 4),
                # DRAM bytes of one evaluation's kernels (ncu capture at configs[2] only)
                "traffic": gmm_traffic() if wl == "gmm" else None,
                "flops_per_eval_survey_W": fl,
                "mat_vec_flops_executed": executed,
                "executed_frac": round(executed / (ms_step * 1e-3) / 1e12 / peak, 4),
                "frac_note": "frac credits SURVEY §8(d)'s W (4 mat-vec passes per point and "
                             "component); executed_frac the 3 passes the kernels execute",
                "peak_source": "max of in-run DMMA m16n8k16 (%.1f TF) and DFMA (%.1f TF) "
                               "microkernels (tools/fp64probe.cu)" % (dmma, dfma)}
    o_ms = D.max(time_device(
        lambda: kernels.gmm_objective(alphas, means, icf, x, gamma, m, cst, N_total=N,
                                      add_param_terms=(D.rank == 0), workspace=ws),
        max(2, min(args.steps // 2, 10)), flush))
    objective = {"ms_per_step": round(o_ms, 4), "grad_over_objective": round(ms_step / o_ms, 3),
                 "kernel": "k_gmm_prep/fwd/lse/err (rl_gmm_objective_f64)"}
    restore = None
    if single:
        restore = {"resid": float(r.resid.item()), "restore_code": int(r.restore_code.item()),
                   "tol": 1e-9, "kernel": "k_gmm_restore (err! chain replayed bit-exactly, "
                                         "side stream beside k_gmm_rev)"}
    res = {
        "metric": "gradient evals/sec", "value": round(1e3 / ms_step, 3), "unit": "evals/s",
        "n_gpus": D.world, "steps": steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": gmm_data(seed),
        "config": dict(gmm_config(d, K, N, D.world), cuda_graph=graph is not None),
        "roofline": roof, "gpu_launches": (6 if single else 5) * steps, "clocks": clocks,
        "failed_per_step": n_failed, "objective_only": objective, "restoration": restore,
    }
    if not args.no_e2e:
        res["e2e"] = gmm_e2e(alphas, means, icf, x, gamma, m, cst, args, D, N)
    return res


def gmm_e2e(alphas, means, icf, x, gamma, m, cst, args, D, N_total):
    """The drop-in gradient through the C-ABI host-buffer entries, pinned host
    inputs up and the packed gradient down inside the timed region.  One GPU:
    rl_gmm_gradient_f64_host (the restoration residual comes down too).  N
    GPUs: each rank rl_gmm_grad_shard_f64_host over its points, then the packed
    vector's sum-allreduce over NCCL (staged through the device) back to host;
    the time is the max over ranks."""
    import ctypes

    import torch

    from paper_2003_04617_b200 import _native
    L = _native.lib()
    K, d = means.shape
    N = x.shape[0]
    single = D.dist is None
    ha, hm, hi_ = alphas.cpu().pin_memory(), means.cpu().pin_memory(), icf.cpu().pin_memory()
    hx = x.cpu().pin_memory()
    nout = 1 + K + K * d + K * d * (d + 1) // 2
    out = torch.empty(nout, dtype=torch.float64).pin_memory()
    stage = torch.empty(nout, dtype=torch.float64, device=x.device)
    nf = ctypes.c_ulonglong()
    resid = ctypes.c_double()

    def call():
        if single:
            rc = L.rl_gmm_gradient_f64_host(d, K, N, ha.data_ptr(), hm.data_ptr(),
                                            hi_.data_ptr(), hx.data_ptr(), gamma, m, cst, 0.0,
                                            1e-9, 1, out.data_ptr(), ctypes.byref(resid),
                                            ctypes.byref(nf), D.gpu)
            if _native.check(rc, "rl_gmm_gradient_f64_host") not in (0, 5):
                raise RuntimeError(f"rl_gmm_gradient_f64_host: status {rc}")
            return
        rc = L.rl_gmm_grad_shard_f64_host(d, K, N, N_total, ha.data_ptr(), hm.data_ptr(),
                                          hi_.data_ptr(), hx.data_ptr(), gamma, m, cst, 1e-9, 1,
                                          int(D.rank == 0), out.data_ptr(), ctypes.byref(nf),
                                          D.gpu)
        _native.check(rc, "rl_gmm_grad_shard_f64_host")
        stage.copy_(out, non_blocking=True)
        D.dist.all_reduce(stage)
        out.copy_(stage)

    call()
    D.barrier()
    t0 = time.perf_counter()
    call()
    one = D.max(time.perf_counter() - t0)
    steps = int(min(50, max(3, 0.3 // max(one, 1e-6))))
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = D.max((time.perf_counter() - t0) / steps)
    h2d = int(hx.numel() * 8 + (ha.numel() + hm.numel() + hi_.numel()) * 8)
    d2h = int(out.numel() * 8 + 32)
    if not single:
        h2d += nout * 8                     # the packed shard vector staged for NCCL
    h2d, d2h = int(D.sum(h2d)), int(D.sum(d2h))   # whole job, like the other arms
    return {"value": round(1.0 / dt, 3), "unit": "evals/s", "calls_timed": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 3),
            "path": ("rl_gmm_gradient_f64_host (pinned host buffers; device buffers and "
                     "workspace carved from a per-thread cached arena, cached streams)" if single
                     else "per rank rl_gmm_grad_shard_f64_host over its points (pinned host "
                          "buffers) + NCCL sum-allreduce of the packed gradient; max over ranks")}


def gmm_cpu(wl, N_full, target_s=1.0):
    """The C oracle (the reference's algorithm: all four sweeps, 8 mat-vec
    passes per point and component, its scratch shared across the points of
    a call) over all host threads: T threads each run it on their own chunk
    of n points (one call per chunk: the shard a data-parallel CPU run would
    give each core; ctypes releases the GIL), n grown until the wall time
    reaches ~target_s; evals/s extrapolated linearly in N (the per-point work
    is the same for every point)."""
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    d, K, _, seed = GMM_CFG[wl]
    rng = np.random.default_rng(seed)
    alphas = rng.standard_normal(K)
    means = rng.random((K, d))
    icf = rng.standard_normal((K, d * (d + 1) // 2))
    T = max(1, min(os.cpu_count() or 1, 64))
    n = 2
    with ThreadPoolExecutor(T) as pool:
        while True:
            xs = [rng.random((n, d)) for _ in range(T)]
            cst = gmm_constants(d, K, n, 1.0, 0)
            t0 = time.perf_counter()
            list(pool.map(lambda x: O.gmm_grad(alphas, means, icf, x, 1.0, 0, cst, tol=1e-6), xs))
            dt = time.perf_counter() - t0
            if dt >= target_s or n * T >= N_full:
                break
            n = min(max(1, N_full // T), max(2 * n, int(n * target_s / max(dt, 1e-4))))
    pts = n * T
    per_eval = dt * N_full / pts
    return {"value": round(1.0 / per_eval, 8), "unit": "evals/s", "cores": T, "kind": "port",
            "sample": f"{pts} of the {N_full} points (d={d}, K={K}): {T} threads each running "
                      f"the oracle (oracle/revoracle.c, all 4 reference sweeps, 8 mat-vec passes "
                      f"per point and component) on {n} points, {dt:.2f} s wall, extrapolated "
                      f"linearly to N={N_full}",
            "extrapolated": pts < N_full}


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks (one per GPU) and pass its output
    through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_line(args, D):
    """--dry-run: the ours-arm line's plumbing without kernels (CPU tests)."""
    t0 = time.perf_counter()
    D.barrier()
    ms = D.max((time.perf_counter() - t0) * 1e3 / max(args.steps, 1) + 1e-3 * (D.rank + 1))
    return {"metric": "gradient evals/sec", "value": None, "unit": "grads/s",
            "n_gpus": D.world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "dry run (no kernels)",
            "config": bessel_config(args.n or BESSEL_N, D.world), "dry_run": True,
            "ranks_reporting": int(D.sum(1)), "dist": D.nccl_info()}


def reference_arm(args, world):
    """The reference algorithm's CPU implementation (the oracle port) on the
    same workloads / configs as the ours arm; bounded samples."""
    # all host threads for the oracle port (torchrun exports OMP_NUM_THREADS=1;
    # libgomp reads it when liboracle.so loads, which happens below)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    tgt = max(2.0, min(20.0, 0.5 * args.steps))
    common = {"n_gpus": world, "steps": args.steps, "warmup": args.warmup,
              "higher_is_better": True, "vs_baseline": None, "dtype": "f64", "impl": "reference",
              "rate_sample": True}

    def line(metric, base, unit, data, config):
        r = {"metric": metric, "value": base["value"], "unit": unit,
             "ms_per_step": round(1e3 / base["value"], 3) if unit != "grads/s" else
             round(1e3 * config["n_total"] / base["value"], 3),
             "scaling": "strong", "data": data, "config": config, "cpu_baseline": base,
             "e2e": {"value": base["value"], "unit": unit, "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0}}
        r.update(common)
        return r

    def bessel():
        return line("gradient evals/sec", bessel_cpu(target_s=tgt), "grads/s",
                    "synthetic z ~ U(0.1, 10), seed 1", bessel_config(args.n or BESSEL_N, world))

    def ba():
        return line("Jacobian evals/sec", ba_cpu(target_s=tgt), "jacobians/s",
                    "synthetic ba20-shaped problem, seed 3", ba_config(args.n or BA_P, world))

    def gmm(wl):
        d, K, N, seed = GMM_CFG[wl]
        N = args.n or N
        return line("gradient evals/sec", gmm_cpu(wl, N), "evals/s", gmm_data(seed),
                    gmm_config(d, K, N, world))

    if args.workload == "all":
        res = bessel()
        res["ba"] = ba()
        res["gmm_c3"] = gmm("gmm")
        res["gmm_c5"] = gmm("gmm_large")
        return res
    if args.workload == "bessel":
        return bessel()
    if args.workload == "ba":
        return ba()
    return gmm(args.workload)


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(reference_arm(args, world)))
        return 0

    D = Dist("gloo" if args.dry_run else args.dist_backend)
    if args.dry_run:
        res = dry_line(args, D)
    else:
        cpu = D.rank == 0 and D.world == 1 and not args.no_cpu_baseline
        if args.workload in ("all", "bessel"):
            res = run_bessel_ours(args, D)
            if cpu:
                res["cpu_baseline"] = bessel_cpu()
        if args.workload in ("all", "ba"):
            r = run_ba_ours(args, D)
            if cpu:
                r["cpu_baseline"] = ba_cpu()
            res = r if args.workload == "ba" else res
            if args.workload == "all":
                res["ba"] = r
        for wl, key in (("gmm", "gmm_c3"), ("gmm_large", "gmm_c5")):
            if args.workload in ("all", wl):
                r = run_gmm_ours(args, D, wl)
                if cpu:
                    r["cpu_baseline"] = gmm_cpu(wl, r["config"]["N"])
                if args.workload == "all":
                    res[key] = r
                else:
                    res = r
        res["dist"] = D.nccl_info()
    if D.rank == 0:
        print(json.dumps(res))
    D.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
