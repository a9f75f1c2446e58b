"""Benchmark: fused PCG32 -> approximate-Gaussian ICDF on B200 (BASELINE.json config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch: 2^28 float32 samples per
GPU from PCG32 (seed 42, stream 0; rank r owns outputs [r 2^28, (r+1) 2^28)),
mapped through the 16-octave x 8-sub-interval piecewise-linear inverse-CDF
table and written to HBM with 128-bit coalesced stores.  Multi-GPU is weak
scaling with no data-path collective (torchrun, one process per GPU, NCCL
only for the barrier and the max-over-ranks time).  Prints ONE JSON line.

``--impl reference`` times the reference's CPU path for the same workload on
the host cores instead: the C restatement in oracle/ (PCG32 + the same
octave x sub-interval evaluator; the reference's own kernels cannot index
sub-intervals), all host threads, bounded samples per step.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BYTES_PER_SAMPLE = 4  # algorithmic: one f32 store, PRNG state in registers
# BASELINE.json "metric" verbatim; `value` is the whole-job aggregate (= per GPU at N=1),
# the HBM-roofline fraction is in `roofline`, MLMC paths/s in `mlmc`.
METRIC = "approx-Gaussian ICDF samples/s per GPU & % HBM roofline; MLMC paths/s"
WORKLOADS = {
    # BASELINE.json configs[1] -- the headline (default)
    "config2": (1 << 28, "subdyadic_linear_k16_s8",
                "config2: PCG32(seed 42, stream 0) -> dyadic piecewise-linear ICDF, 16 octaves x 8 "
                "sub-intervals per tail, degree-1 L2 fit, f32 out, 2^28 samples/GPU/step"),
    # BASELINE.json configs[0] -- the reference's CPU-runnable case
    "config1": (1 << 24, "constant_q10_l1",
                "config1: PCG32(seed 42, stream 0) -> piecewise-constant ICDF, 2^10 equal intervals, "
                "L1 (conditional-mean) values, f32 out, 2^24 samples/GPU/step"),
}
N_PER_GPU, TABLE, WORKLOAD = WORKLOADS["config2"]


def select_workload(name: str) -> None:
    global N_PER_GPU, TABLE, WORKLOAD
    N_PER_GPU, TABLE, WORKLOAD = WORKLOADS[name]


def _peaks() -> dict:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples: list[int] = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                break
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self) -> dict:
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [k for k, bit in self.REASONS.items() if self.reasons & bit and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "n_samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port; the checker is never the measured product)
# ---------------------------------------------------------------------------

def cpu_port_rate(total: int, threads: int) -> tuple[float, float]:
    """samples/s of the oracle's fused PCG32 -> sub-interval evaluator on `threads` host threads."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    c = np.load(os.path.join(REPO, "paper_2012_09715_b200", "data", "tables.npz"))[TABLE].astype(np.float32)
    per = max(4, (total // threads) & ~3)
    chunk = min(per, 1 << 22)  # bounded host memory; each thread writes its range chunk by chunk
    bufs = [np.empty(chunk, dtype=np.float32) for _ in range(threads)]
    cptr = c.ctypes.data_as(oracle.oracle.C.c_void_p)
    vp = oracle.oracle.C.c_void_p

    def work(i):
        o = bufs[i].ctypes.data_as(vp)
        for lo in range(0, per, chunk):
            m = min(chunk, per - lo)
            if TABLE.startswith("constant"):
                oracle.lib.orc_pcg32_constant_f32(42, 0, i * per + lo, cptr, int(np.log2(c.size)), o, m)
            else:
                oracle.lib.orc_pcg32_subdyadic_f32(42, 0, i * per + lo, cptr, 1, 16, 3, o, m)

    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        list(ex.map(work, range(threads)))
        dt = time.perf_counter() - t0
    return per * threads / dt, dt


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(target_seconds: float = 8.0) -> dict:
    threads = cpu_threads()
    r1, _ = cpu_port_rate(1 << 22, threads)  # calibration
    total = int(min(max(r1 * target_seconds, 1 << 22), 1 << 36))
    rate, dt = cpu_port_rate(total, threads)
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "")
    except Exception:
        pass
    return {"value": rate, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{total} samples of the {WORKLOAD.split(':')[0]} workload (oracle/oracle.c PCG32 + the same "
                      f"table evaluator, -O3 generic x86-64, no FMA), {threads} threads, {dt:.2f} s; CPU: {model}"}


def _ref_kernel_worker(args):
    """One process: the reference's compiled dyadic_eval32 (oracle/_ref) on a chunk."""
    offset, n, reps = args
    import oracle

    ref = oracle.load_ref_kernels()
    c = np.load(os.path.join(REPO, "paper_2012_09715_b200", "data", "tables.npz"))["dyadic_linear_k15"]
    c32 = c.astype(np.float32)
    u = oracle.u32_to_f32(oracle.pcg32_words(42, 0, offset, n))
    out = np.empty_like(u)
    ref.dyadic_eval32(c32, u, out)  # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        ref.dyadic_eval32(c32, u, out)
    return n * reps, time.perf_counter() - t0


def reference_kernel_rate(procs: int, n_per_proc: int = 1 << 22, reps: int = 3) -> dict | None:
    """The reference's own Cython kernel (compiled from /root/reference into oracle/_ref),
    dyadic_eval32 on the K15 table over the same PCG32 lattice uniforms, one process
    per core (the Cython loop holds the GIL).  Uniform generation is excluded."""
    import multiprocessing as mp

    import oracle

    if oracle.load_ref_kernels() is None:
        return None
    with mp.get_context("spawn").Pool(procs) as pool:
        res = pool.map(_ref_kernel_worker, [(i * n_per_proc, n_per_proc, reps) for i in range(procs)])
    samples = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": samples / wall, "unit": "samples/s", "cores": procs, "kind": "reference",
            "sample": f"oracle/_ref _kernels.dyadic_eval32 (reference Cython, -O3) on the K15 linear table, "
                      f"{procs} processes x {reps} x {n_per_proc} PCG32 lattice uniforms (generation excluded)"}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args) -> None:
    if int(os.environ.get("RANK", "0")) != 0:
        return
    threads = cpu_threads()
    per_step = min(args.ref_samples, N_PER_GPU)
    for _ in range(max(args.warmup, 0)):
        cpu_port_rate(per_step, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_port_rate(per_step, threads)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (PCG32 stream)",
        "impl": "reference",
        "config": {"workload": WORKLOAD, "samples_per_step": per_step, "note": "bounded sample per step on host"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} samples per step, {threads} threads, oracle/oracle.c"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        rk = reference_kernel_rate(threads)
    except Exception as exc:  # the context figure must never break the arm
        rk = {"unavailable": f"{type(exc).__name__}: {exc}"}
    if rk is not None:
        line["reference_kernel"] = rk
    try:
        line["reference_sampler"] = reference_sampler_rate(threads)
    except Exception as exc:
        line["reference_sampler"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)


def reference_sampler_rate(procs: int, n_per_proc: int = 1 << 24) -> dict | None:
    """The reference's whole sampling path with generation: UniformStream.uniforms
    (numpy Philox-4x64) + eval_dyadic(float32) through its compiled kernel,
    one process per core on disjoint stream ids (oracle/refpath.py)."""
    import oracle
    from oracle import refpath

    if oracle.load_ref_kernels() is None:
        return None
    units, wall = refpath.run_pool(refpath.sampler_path, [(42, j, n_per_proc, 1 << 20) for j in range(procs)],
                                   procs)
    return {"value": units / wall, "unit": "samples/s", "cores": procs, "kind": "reference",
            "sample": f"{procs} processes x {n_per_proc} samples: UniformStream(42, j).uniforms (numpy Philox) -> "
                      f"f32 -> oracle/_ref _kernels.dyadic_eval32 (reference Cython), K15 linear table"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _load_traffic(n: int) -> float | None:
    """DRAM bytes per launch of this workload's kernel from the committed ncu
    capture (profiles/ncu_summary.json, measured at its own sample count and
    scaled per sample), or None."""
    p = os.path.join(REPO, "profiles", "ncu_summary.json")
    key = "constant" if TABLE.startswith("constant") else "subdyadic"
    try:
        with open(p) as fh:
            d = json.load(fh)[key]
        return d["dram_bytes_per_launch"] / d["samples_per_launch"] * n
    except Exception:
        return None


def _fp64_roofline(key: str, path_steps_per_s: float) -> dict | None:
    """FP64 roofline of an MLMC level kernel: achieved = FP64 FLOP per path-step
    (ncu dadd + dmul + 2 dfma of the committed capture, profiles/ncu_summary.json)
    x measured path-steps/s; peak = 64 DFMA lanes/SM/clk x 2 x SMs x max SM clock."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)[key]
        import torch

        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        mhz = _peaks().get("sm_max_mhz", 1965.0)
        peak = 64 * 2 * sms * mhz * 1e6 / 1e12
        achieved = d["dp_flops_per_path_step"] * path_steps_per_s / 1e12
        # DADD/DMUL occupy a DFMA lane for 1 FLOP, so also report FP64 lane-op issue vs the lane peak
        lane_frac = d["dp_lane_ops_per_path_step"] * path_steps_per_s / (64 * sms * mhz * 1e6)
        return {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "fp64_lane_op_frac": lane_frac,
                "flops_per_path_step": d["dp_flops_per_path_step"], "fp64_pipe_active_pct_ncu": d["fp64_pipe_active_pct"],
                "peak_source": "nominal: ncu peak_sustained 64 DFMA/SM/clk x max SM clock (MEASURED_PEAKS sm_max_mhz)"}
    except Exception:
        return None


def time_generator(arv, _native, table, n, offset, steps, device):
    """Per-launch seconds of the fused generator over `steps` launches and the
    launch count.  Outputs smaller than L2 are timed launch by launch with a
    512 MiB store sweep flushing L2 in between (outside the events); larger
    outputs stream straight through L2 and are timed back to back."""
    import torch

    out = torch.empty(n, dtype=torch.float32, device=device)

    def step():
        arv.Pcg32Stream(42, 0, counter=offset).sample(table, n, out=out)

    for _ in range(3):
        step()
    flush = n * 4 < (256 << 20)
    scratch = torch.empty(128 << 20, dtype=torch.float32, device=device) if flush else None
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    if flush:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        s = torch.cuda.current_stream().cuda_stream
        for a, b in evs:
            _native.call("arv_store_probe", scratch.data_ptr(), scratch.numel(), s)
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
        elapsed = sum(a.elapsed_time(b) for a, b in evs) * 1e-3
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            step()
        b.record()
        b.synchronize()
        elapsed = a.elapsed_time(b) * 1e-3
    launches = _native.launch_count() - l0 - (steps if flush else 0)
    return elapsed / steps, launches, flush


def config1_entry(arv, _native, device, offset: int, peak: float, steps: int = 200) -> dict:
    """BASELINE configs[0] (2^24 samples, piecewise-constant q=10 table) on the
    same GPU: per-launch time with L2 flushed between launches, HBM roofline."""
    n, tname, wl = WORKLOADS["config1"]
    per_launch, launches, _ = time_generator(arv, _native, arv.load_table(tname), n, offset, steps, device)
    achieved = n * BYTES_PER_SAMPLE / per_launch / 1e9
    # the same protocol for a store-only kernel of the same size: what a pure
    # 64 MiB write achieves per launch (launch + ramp + drain included)
    import torch

    out = torch.empty(n, dtype=torch.float32, device=device)
    scratch = torch.empty(128 << 20, dtype=torch.float32, device=device)
    s = torch.cuda.current_stream().cuda_stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in evs:
        _native.call("arv_store_probe", scratch.data_ptr(), scratch.numel(), s)
        a.record()
        _native.call("arv_store_probe", out.data_ptr(), n, s)
        b.record()
    torch.cuda.synchronize()
    probe = sum(a.elapsed_time(b) for a, b in evs) * 1e-3 / len(evs)
    # the same event sandwich around an (almost) empty launch: the fixed cost inside every figure above
    for a, b in evs:
        _native.call("arv_store_probe", scratch.data_ptr(), scratch.numel(), s)
        a.record()
        _native.call("arv_store_probe", out.data_ptr(), 8, s)
        b.record()
    torch.cuda.synchronize()
    empty = sum(a.elapsed_time(b) for a, b in evs) * 1e-3 / len(evs)
    # Back to back without the per-launch event pair: a CUDA graph of 16 launches over a ring of
    # 8 output buffers (512 MiB > L2: no launch writes lines the previous ones left in L2);
    # programmatic dependent launch overlaps each launch's start-state walk with the previous tail.
    table = arv.load_table(tname)
    ring = [torch.empty(n, dtype=torch.float32, device=device) for _ in range(8)]
    side = torch.cuda.Stream(device=device)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(8):
            arv.Pcg32Stream(42, 0, counter=offset).sample(table, n, out=ring[i])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(16):
                arv.Pcg32Stream(42, 0, counter=offset + i * n).sample(table, n, out=ring[i % 8])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            g.replay()
        b.record()
        b.synchronize()
        ring_t = a.elapsed_time(b) * 1e-3 / 160
    torch.cuda.current_stream().wait_stream(side)
    ring_bw = n * BYTES_PER_SAMPLE / ring_t / 1e9
    return {"workload": wl, "value": n / per_launch, "unit": "samples/s", "us_per_launch": per_launch * 1e6,
            "steps": steps, "gpu_launches": int(launches),
            "l2": "output < L2: each launch timed alone, 512 MiB store sweep flushes L2 in between",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "algorithmic_bytes_per_launch": n * BYTES_PER_SAMPLE,
                         "store_probe_same_size_us": probe * 1e6,
                         "frac_of_store_probe_same_size": probe / per_launch,
                         "empty_launch_same_protocol_us": empty * 1e6},
            "back_to_back": {"us_per_launch": ring_t * 1e6, "value": n / ring_t, "unit": "samples/s",
                             "achieved": ring_bw, "frac": ring_bw / peak, "gpu_launches": 160,
                             "l2": "ring of 8 output buffers (512 MiB > L2), 10 replays of a CUDA graph of 16 launches, "
                                   "one event pair around all of them"}}


def e2e_plugin(arv, device, steps: int = 3) -> dict:
    """The reference's calling convention end to end: the drop-in plugin call
    ``_kernels.dyadic_eval32(coeffs32, u, out)`` (_kernels.pyx:76-93) on 2^28
    numpy f32 uniforms into a caller-allocated numpy out -- H2D of u, kernel,
    D2H into out inside the timed region (host-buffer pipeline,
    csrc/arv_host.cu).  Same work as `reference_kernel` in the reference arm."""
    import torch

    from paper_2012_09715_b200 import _kernels

    n = 1 << 28
    lin = arv.load_table("dyadic_linear_k15")
    u = arv.Pcg32Stream(42, 0).uniforms(n).cpu().numpy()  # the lattice uniforms, host
    out = np.empty(n, np.float32)
    out.fill(0.0)  # pages touched once (as the reference's np.empty_like + its own writes)
    _kernels.dyadic_eval32(lin.coeffs32, u[: 1 << 20], out[: 1 << 20])  # warm (pinned staging allocated)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        _kernels.dyadic_eval32(lin.coeffs32, u, out)  # returns when out is written
    dt = (time.perf_counter() - t0) / steps
    ref = arv.eval_dyadic(lin, torch.from_numpy(u[: 1 << 16]).to(device), dtype=np.float32).cpu().numpy()
    assert np.array_equal(out[: 1 << 16].view(np.uint32), ref.view(np.uint32))
    return {"value": n / dt, "unit": "samples/s", "h2d_bytes_per_step": n * 4, "d2h_bytes_per_step": n * 4,
            "ms_per_step": dt * 1e3, "samples_per_step": n,
            "path": "paper_2012_09715_b200._kernels.dyadic_eval32(numpy f32 u, numpy f32 out), K15 linear table: "
                    "pinned-chunk pipeline (host copies || H2D || kernel || D2H), host wall clock"}


def shard_check(out, rank: int, world: int, device) -> dict:
    """Sum of the shard's 64-bit words mod 2^64 on the device, against the
    oracle's value for this rank's offset range (tests/golden/hashes.json)."""
    import torch

    s = int(out.view(torch.int64).sum().item()) % (1 << 64)
    try:
        with open(os.path.join(REPO, "tests", "golden", "hashes.json")) as fh:
            want = json.load(fh).get("config2_shard_word_sums_mod2^64", [])
        ok = (str(s) == want[rank]) if rank < len(want) and N_PER_GPU == 1 << 28 else None
    except Exception:
        ok = None
    t = torch.tensor([rank, 1 if ok else (0 if ok is False else -1)], dtype=torch.int64, device=device)
    if world > 1:
        import torch.distributed as dist

        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        flags = [int(g[1].item()) for g in got]
        backend = dist.get_backend()
    else:
        flags, backend = [int(t[1].item())], None
    return {"ranks": world, "backend": backend, "rank_ok": flags, "all_match": all(f == 1 for f in flags),
            "check": "per-rank sum of output words mod 2^64 vs the oracle's for its PCG32 offset range"}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # ARV_BENCH_DIST_BACKEND=gloo exercises the multi-rank code path on a box
        # with fewer GPUs (ranks share devices; gloo syncs on the host, so no GPU
        # kernel ever waits on another rank).  Production runs use NCCL.
        backend = os.environ.get("ARV_BENCH_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    device = torch.device("cuda", torch.cuda.current_device())

    import paper_2012_09715_b200 as arv
    from paper_2012_09715_b200 import _native

    table = arv.load_table(TABLE)
    n = N_PER_GPU
    out = torch.empty(n, dtype=torch.float32, device=device)
    offset = rank * n

    def step():
        arv.Pcg32Stream(42, 0, counter=offset).sample(table, n, out=out)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(device.index)
    # Outputs smaller than L2 (config 1: 64 MiB) are timed launch by launch
    # with a 512 MiB store sweep flushing L2 between launches (outside the
    # events); larger outputs stream straight through L2.
    flush = n * 4 < (256 << 20)
    scratch = torch.empty(128 << 20, dtype=torch.float32, device=device) if flush else None
    barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    elapsed = 0.0
    with sampler:
        if flush:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            s = torch.cuda.current_stream().cuda_stream
            for a, b in evs:
                _native.call("arv_store_probe", scratch.data_ptr(), scratch.numel(), s)
                a.record()
                step()
                b.record()
            torch.cuda.synchronize()
            elapsed = sum(a.elapsed_time(b) for a, b in evs) * 1e-3
        else:
            start.record()
            for _ in range(args.steps):
                step()
            stop.record()
            stop.synchronize()
            elapsed = start.elapsed_time(stop) * 1e-3
    launches = _native.launch_count() - l0 - (args.steps if flush else 0)
    barrier()
    torch.cuda.synchronize()
    t = torch.tensor([elapsed], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = world * n * args.steps / t_max
    per_launch = t_max / args.steps

    # approximation quality of this step's output (untimed): error against the
    # exact AS241 f64 quantile of the same uniforms, over every sample
    quality = approximation_error(arv, out, offset)
    shards = shard_check(out, rank, world, device)

    # e2e: the public API with a pinned host buffer, D2H inside the timed region
    host = torch.empty(n, dtype=torch.float32, pin_memory=True)
    arv.Pcg32Stream(42, 0, counter=offset).sample_host(table, n, out=host)  # warm
    e_steps = max(1, min(args.steps, 5))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e_steps):
        arv.Pcg32Stream(42, 0, counter=offset).sample_host(table, n, out=host, sync=False)
    e1.record()
    e1.synchronize()
    et = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = world * n * e_steps / float(et.item())

    # store-only roof of this GPU (same output buffer, st.global.v4 of a constant)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        _native.call("arv_store_probe", out.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    s0.record()
    for _ in range(20):
        _native.call("arv_store_probe", out.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    s1.record()
    s1.synchronize()
    store_gbs = n * 4 * 20 / (s0.elapsed_time(s1) * 1e-3) / 1e9

    mlmc = None if args.no_mlmc else mlmc_metrics(arv, args, rank, world, device)
    peak = _peaks().get("hbm_gbs") or 6650.0
    c1 = config1_entry(arv, _native, device, rank * WORKLOADS["config1"][0], peak) \
        if N_PER_GPU != WORKLOADS["config1"][0] else None
    plugin = e2e_plugin(arv, device) if rank == 0 and not args.no_plugin else None

    # sustained (last GPU phase, so the power ramp cannot slow the MLMC timings):
    # the same launches back to back for ~2 s; the second half is
    # past the board's power ramp (the generator reaches the power cap)
    sustained = None
    if not args.no_sustained:
        sus_s, sus_clocks = sustained_per_launch(step, device, seconds=2.0)
        st = torch.tensor([sus_s], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(st, op=dist.ReduceOp.MAX)
        sustained = {"value": world * n / float(st.item()), "unit": "samples/s",
                     "us_per_launch": float(st.item()) * 1e6, "window": "launches in t = 1..2 s of a 2 s run",
                     "clocks": sus_clocks}


    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = _peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs, copy)" if peak else "fallback (B200_PROFILING.md 6.65 TB/s)"
    peak = peak or 6650.0
    achieved = n * BYTES_PER_SAMPLE / per_launch / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (PCG32 stream, no dataset)",
        "config": {"workload": WORKLOAD, "table": TABLE, "samples_per_gpu_per_step": n,
                   "parallelism": f"dp{world} (PCG32 offset shards, no data-path collective)",
                   "l2": ("output 1 GiB per GPU per step > 126 MB L2 (no flush needed)" if n * 4 >= (256 << 20) else
                          "output < L2: each launch timed alone, 512 MiB store sweep flushes L2 in between")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _load_traffic(n), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": n * BYTES_PER_SAMPLE,
                     "store_only_probe_gbs": store_gbs, "frac_of_store_probe": achieved / store_gbs},
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": n * 4,
                "path": "Pcg32Stream.sample_host -> pinned host buffer, chunked D2H overlapped with generation"},
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
        "quality": quality,
        "sustained": sustained,
        "shard_check": shards,
    }
    if plugin is not None:
        line["e2e_plugin"] = plugin
    if c1 is not None:
        line["config1"] = c1
    if mlmc is not None:
        line["mlmc"] = mlmc
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sustained_per_launch(step, device, seconds: float = 2.0, window: int = 25):
    """Mean per-launch time over the second half of `seconds` of back-to-back
    launches (CUDA events per window of `window` launches), with NVML clocks."""
    import torch

    sampler = ClockSampler(device.index)
    done, tail = 0.0, []
    with sampler:
        while done < seconds:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(window):
                step()
            b.record()
            b.synchronize()
            dt = a.elapsed_time(b) * 1e-3
            done += dt
            if done > seconds / 2:
                tail.append(dt / window)
    return statistics.mean(tail), sampler.summary()


def approximation_error(arv, out, offset: int, chunk: int = 1 << 26) -> dict:
    """RMSE / max |error| of the f32 table samples against AS241 in f64 on the
    same PCG32 uniforms, all samples of one step."""
    import torch

    n = out.numel()
    sq, mx = 0.0, 0.0
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        ex = arv.Pcg32Stream(42, 0, counter=offset + lo).sample_exact64(m)
        d = out[lo:lo + m].double() - ex
        sq += float(torch.dot(d, d))
        mx = max(mx, float(d.abs().max()))
    return {"rmse_vs_as241_f64": math.sqrt(sq / n), "max_abs_err": mx, "samples": n,
            "note": "table approximation error, not a parity measure (parity is bit-exact, tests/)"}


def mlmc_metrics(arv, args, rank, world, device) -> dict:
    """Config 4 (GBM EM, l=0..8, 2^22 paths/level) and config 5 (CIR exact, l=0..6,
    2^20 paths/level): one full multilevel pilot through the public estimator
    ``estimate_level_suites`` (estimate_level_suite, mlmc.py:383-411, for all
    levels).  At N > 1 each level's paths are sharded over the ranks and the
    (count, mean, M2) triples of all levels and the failure count are merged by
    NCCL all-reduces (mlmc.allreduce_triples), so the reported statistics are
    the whole job's.  Timed with CUDA events around the whole pilot (host work
    included), max over ranks."""
    import torch

    from paper_2012_09715_b200 import _native

    group = None
    if world > 1:
        import torch.distributed as dist

        group = dist.group.WORLD
    res = {}
    lin = arv.load_table("dyadic_linear_k15")
    cases = [
        ("gbm_em_config4", arv.GbmParams(0.05, 0.2, 1.0, 1.0), "euler_maruyama", lin, range(0, 9), 1 << 22),
        ("cir_exact_config5", arv.CirParams(0.5, 0.04, 0.2, 0.04, 1.0), "cir_exact",
         arv.load_table("ncchi2_cir_k64_stacks"), range(0, 7), 1 << 20),
    ]
    for name, proc, scheme, tab, levels, n_paths in cases:
        specs = [arv.LevelSpec(level=l, scheme=scheme, process=proc, rv_source=tab, kind="four_way", n0=1)
                 for l in levels]
        streams = [arv.level_stream(42, sp.level) for sp in specs]
        # warm-up: one untimed full pilot (workspace allocations, module loads)
        arv.estimate_level_suites(specs, streams, n_paths, group=group)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        certified = ctypes.c_ulonglong(0)
        if scheme == "cir_exact":
            _native.call("arv_nc_certified_count", ctypes.byref(certified))  # reset (outside the timed region)
        e0.record()
        # raises NumericalError if any rank's exact transitions failed
        suites = arv.estimate_level_suites(specs, streams, n_paths, group=group)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t.item())
        steps = sum(1 << l for l in levels)
        paths_total = n_paths * len(levels)
        entry = {"paths_per_level": n_paths, "levels": [levels[0], levels[-1]], "seconds": secs,
                 "paths_per_s": paths_total / secs, "path_steps_per_s": n_paths * steps / secs,
                 "api": "estimate_level_suites (all levels back to back, one host sync)" +
                        (f"; one {dist.get_backend().upper()} all-reduce pair of all levels' triples over {world} ranks"
                         if world > 1 else "")}
        entry["roofline"] = _fp64_roofline("gbm_level8" if scheme != "cir_exact" else "cir_level6",
                                           n_paths * steps / secs)
        if scheme == "cir_exact":
            entry["n_fail"] = 0
            # exact transitions solved with one CDF sweep (certified Taylor root, csrc/arv_ncchi2.cuh)
            _native.call("arv_nc_certified_count", ctypes.byref(certified))
            my_paths = suites[0][next(iter(suites[0]))].n_paths // max(world, 1)
            entry["single_sweep_solves_share"] = int(certified.value) / max(my_paths * steps, 1)
            entry["log2_correction_gap"] = [float(np.log2(s["correction"].variance / s["plain_exact"].variance))
                                            for s in suites]
            entry["process_variance"] = [s["plain_exact"].variance for s in suites]
        else:
            entry["log2_four_way_gap"] = [float(np.log2(s["four_way"].variance / s["two_way_exact"].variance))
                                          for s in suites[1:]]
            entry["level0_mean"] = suites[0]["two_way_exact"].mean
        entry["n_paths_merged"] = [s[next(iter(s))].n_paths for s in suites]
        if world == 1 and rank == 0 and not args.no_cpu:
            entry["cpu_baseline"] = mlmc_cpu_baseline(name, levels, n_paths)
        res[name] = entry
    return res


def mlmc_cpu_baseline(name: str, levels, n_paths: int, budget_s: float = 10.0) -> dict:
    """The reference's MLMC pilot on the host cores (oracle/refpath.py: the C
    restatement of simulate_gbm_coupled / the numpy-scipy restatement of
    simulate_cir_coupled(cir_exact), one process per core), on a bounded
    sample of the same levels: a fraction f of each level's paths, f sized from
    a calibration run to ~budget_s of wall time."""
    from oracle import refpath

    procs = cpu_threads()
    if name.startswith("gbm"):
        fn, make = refpath.gbm_level, (lambda l, m, j: (l, n_paths, j * m, (j + 1) * m))
        kind_note = "oracle.c orc_gbm_paths (C restatement of simulate_gbm_coupled, -O3, no FMA)"
    else:
        fn, make = refpath.cir_exact_level, (lambda l, m, j: (l, m, 42 + j))
        kind_note = "oracle/cir.py (numpy/scipy restatement of simulate_cir_coupled cir_exact, CDFLIB chndtr)"
    cal_units, cal_wall = refpath.run_pool(fn, [make(levels[-1], 256, j) for j in range(procs)], procs)
    rate0 = cal_units / cal_wall
    total = n_paths * sum(1 << l for l in levels)
    f = min(1.0, rate0 * budget_s / total)
    m = max(16, int(n_paths * f) // procs)
    jobs = [make(l, m, j) for l in levels for j in range(procs)]
    units, wall = refpath.run_pool(fn, jobs, procs)
    return {"value": units / wall, "unit": "path-steps/s", "cores": procs, "kind": "port",
            "paths_per_s": m * procs * len(levels) / wall,
            "seconds_full_config_extrapolated": total / (units / wall),
            "sample": f"{m * procs} paths per level x levels {levels[0]}..{levels[-1]} ({units} path-steps, "
                      f"{wall:.1f} s wall), {procs} processes; {kind_note}"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-mlmc", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-plugin", action="store_true")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="config2")
    ap.add_argument("--ref-samples", type=int, default=1 << 28,
                    help="reference arm: bounded host sample per step (samples)")
    args = ap.parse_args()
    select_workload(args.workload)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
