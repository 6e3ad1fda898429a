#!/usr/bin/env python
"""Benchmark of the hot path: suffix-array build (Msuffixes/s) + overlap queries/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c1..c5] [--sweep]

One "step" = one complete SA build (2-bit pack, k-mer initial sort, prefix-doubling rounds)
over the synthetic read text of the named BASELINE.json configuration.  Prints ONE JSON line.

  value    : n_suffixes * steps / device time, text already resident in HBM (CUDA events on
             the launching stream, max over ranks)
  e2e      : the same build through the host-buffer C-ABI call reseq_cuda_build_sa (pinned
             host text in, sa + rank out to pinned host buffers; H2D and D2H inside the timed
             region)
  roofline : the dominant kernel (one onesweep digit pass over (u64 key, u32 position) pairs),
             timed live with CUDA events around every launch inside the timed region
  cpu_baseline : the reference's own build_parallel (oracle/_ref) on a bounded prefix of the
             same text, on this box's host cores
  routes   : the same text through the two general engines (general DNA records: what a ragged read
             set takes; prefix doubling: the north star's algorithm), forced by context options
  overlap  : the batched SA search job (queries/s) measured after the timed steps, with its own
             roofline (per-kernel CUDA-event times, ncu DRAM bytes from profiles/), e2e and the
             reference's locate_prefix_range loop on this box's host cores as cpu_baseline
  sweep    : (--sweep, or --workload c3) SA build throughput over n = 2^20 .. full by truncating k

`--impl reference` times the reference CPU implementation only (no GPU work).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (genome bases, read length, reads) -- SURVEY.md section 8(d) / BASELINE.md section 3
    "c1": (1_000_000, 100, 100_000),
    "c2": (4_600_000, 150, 920_000),
    "c3": (10_000_000, 150, 666_666),
    "c4": (100_000_000, 150, 6_666_666),
    "c5": (300_000_000, 150, 20_000_000),
}
DESCRIPTION = {
    "c1": "config[0]: 1 Mbp genome, 100-bp reads, 10x (n=10.1M suffixes)",
    "c2": "config[1]: 4.6 Mbp genome, 150-bp reads, 30x (n=138.92M suffixes)",
    "c3": "config[2]: 100 Mbp concatenated read text (n=100.67M suffixes)",
    "c4": "config[3]: 1 Gbp read set (n=1.0067G suffixes)",
    "c5": "config[4]: 3 Gbp human-scale read set (n=3.02G suffixes; beyond the reference's 2^31-1 cap)",
}
METRIC = "sa_build_msuffixes_per_s"
UNIT = "Msuffixes/s"


def bytes_alg_per_suffix(n: int, read_len: int) -> tuple[float, int, int]:
    """80 + R16*(44 + 24*P) + 8 with P = ceil(2*ceil(log2(n+2))/8)."""
    b = int(np.ceil(np.log2(n + 2)))
    P = -(-2 * b // 8)
    R16 = int(np.ceil(np.log2(np.ceil((read_len + 1) / 16))))
    return 80 + R16 * (44 + 24 * P) + 8, P, R16


def measured_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._pump, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- reference / CPU baseline ------------------------------------------------------------

def _load_cpu_lib():
    """oracle/_ref (the real reference) if present, else the oracle port.  The only place
    bench.py touches oracle/: the CPU baseline, never the measured product path."""
    ref = ROOT / "oracle" / "_ref" / "libreseq_ref.so"
    if ref.exists():
        try:
            return C.CDLL(str(ref)), "reference"
        except OSError:
            pass
    port = ROOT / "oracle" / "liboracle.so"
    if not port.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    return C.CDLL(str(port)), "port"


def cpu_read_text(G: int, L: int, k: int) -> np.ndarray:
    """The first k reads of the SURVEY 8(d) text, generated by the CPU libraries (reads are drawn one
    after another from one RNG stream, so a prefix of the reads is a prefix of the text)."""
    lib, kind = _load_cpu_lib()
    out = np.empty(k * (L + 1), np.uint8)
    fn = lib.ref_make_read_text if kind == "reference" else lib.orc_make_read_text
    st = fn(C.c_size_t(G), C.c_size_t(L), C.c_size_t(k), C.c_uint64(1), C.c_uint64(2), out.ctypes.data_as(C.c_void_p))
    if st != 0:
        raise RuntimeError("CPU text generator failed")
    return out


def cpu_build(lib, kind: str, text: np.ndarray, workers: int) -> float:
    """One reference build_parallel (or oracle build) of `text`; returns seconds."""
    n = text.size
    sa = np.empty(n, np.uint32)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    t0 = time.perf_counter()
    if kind == "reference":
        st = lib.ref_build_parallel(vp(text), C.c_size_t(n), C.c_uint(workers), C.c_size_t(1 << 15), vp(sa), None)
    else:
        st = lib.orc_build_sa(vp(text), C.c_size_t(n), vp(sa), None)
    dt = time.perf_counter() - t0
    if st != 0:
        raise RuntimeError("CPU baseline build failed")
    return dt


def cpu_sample(text: np.ndarray, read_len: int, target_bytes: int) -> np.ndarray:
    reads = max(1, min(text.size, target_bytes) // (read_len + 1))
    return np.ascontiguousarray(text[: reads * (read_len + 1)])


def run_reference(args, text, read_len, workload):
    lib, kind = _load_cpu_lib()
    cores = os.cpu_count() or 1
    workers = cores if kind == "reference" else 1
    steps, warmup = args.steps, args.warmup
    # calibrate the sample so that (steps + warmup) builds end within ~150 s
    probe = cpu_sample(text, read_len, 1 << 17)
    t_probe = cpu_build(lib, kind, probe, workers)
    # build_parallel is ~n log^2 n: time(n) ~ t_probe * (n / n_probe)^1.35 measured here; solve for the budget
    budget = 120.0 / max(1, steps + warmup)
    target = int(min(1 << 22, max(1 << 16, probe.size * (budget / t_probe) ** (1 / 1.35))))
    sample = cpu_sample(text, read_len, target)
    for _ in range(warmup):
        cpu_build(lib, kind, sample, workers)
    t = [cpu_build(lib, kind, sample, workers) for _ in range(steps)]
    total = float(sum(t))
    value = sample.size * steps / total / 1e6
    desc = (f"first {sample.size // (read_len + 1)} reads ({sample.size} suffixes) of the {workload} text; "
            f"{'reference build_parallel (suffix_array.hpp:61), executor{workers=' + str(workers) + ', chunk=32768}' if kind == 'reference' else 'oracle port (std::sort on suffix order), 1 thread'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": total / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": DESCRIPTION[workload], "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# B/suffix one launch of each kernel accounts for in the SURVEY 8(d) model.  The refine kernel
# stands for ALL doubling rounds of the model (R16 * (44 + 24 P)): it reaches the same order by
# fetching keys from the L2-resident packed text, so its figure can exceed the HBM peak -- its
# real DRAM traffic is in `traffic` (ncu).  The partition passes + window scatter stand for the
# model's inverse-permutation phase (8 B/suffix) and are listed with their own minimal traffic.
KERNEL_MODEL_BYTES = {
    "pack_dna_kernel": 1.375, "initkey_dna_kernel": 8.375, "initkey_bytes_kernel": 9.0,
    "onesweep_u32_pairs": 16.0, "onesweep_u32_keys": 8.0, "onesweep_u64_pairs": 24.0,
    "init_elems_kernel": 8.375, "onesweep_u64_keys": 16.0,
    "refine_elems_kernel": 13.4, "window_scatter_kernel": 12.0, "inv_partition_sa": 12.0, "inv_partition_rec": 16.0,
    "inv_partition_rec0": 16.0, "inv_partition_sa_val": 16.0,
    "inverse_kernel": 8.0, "pair_key_kernel": 20.0, "rerank_kernel": 16.0, "hist_kernel": 4.0,
    "gen_uniform_kernel": 8.25, "accept_uniform_kernel": 12.25,   # link / refine touch a few % of the suffixes: no figure
    "owner_partition_kernel": 12.0, "owner_count_kernel": 4.0,
}


def ncu_sa_traffic(workload: str) -> dict:
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the SA kernels from the ncu --set full
    captures under profiles/ (r2_ncu_sa_traffic.json: {workload: {kernel: bytes}})."""
    p = ROOT / "profiles" / "r2_ncu_sa_traffic.json"
    if p.exists():
        try:
            return {k: float(v) for k, v in json.loads(p.read_text()).get(workload, {}).items()}
        except Exception:
            pass
    return {}


def roofline_block(prof: dict, n: int, L: int, steps: int, ms_per_step: float, workload: str, n_kernel: int = None) -> dict:
    """`prof` = {kernel: (launches, total ms)} over `steps` steps; n_kernel = suffixes one launch
    processes when that is not n (a multi-GPU rank's bucket)."""
    peak, peak_src = measured_peak()
    per_suffix, P, R16 = bytes_alg_per_suffix(n, L)
    nk = n_kernel or n
    ncu_traffic = ncu_sa_traffic(workload)
    kernels = {}
    for kname, (cnt, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        b = KERNEL_MODEL_BYTES.get(kname)
        avg = ms / cnt if cnt else None
        ach = b * nk / (avg * 1e-3) / 1e9 if (b and avg) else None
        kernels[kname] = {"ms_per_step": ms / steps, "launches_per_step": cnt / steps,
                          "avg_launch_ms": avg, "alg_bytes_per_suffix": b,
                          "achieved_gbs": ach, "frac": ach / peak if ach else None,
                          "share_of_step": (ms / steps) / ms_per_step}
    dom_name = next(iter(kernels)) if kernels else "none"
    dom = kernels.get(dom_name, {})
    kernel_ms = sum(v[1] for v in prof.values()) / steps
    return {
        "bound": "hbm", "kernel": dom_name, "achieved": dom.get("achieved_gbs"), "peak": peak, "unit": "GB/s",
        "frac": dom.get("frac"), "traffic": ncu_traffic.get(dom_name),
        "peak_source": peak_src,
        "alg_bytes_per_launch": (dom.get("alg_bytes_per_suffix") or 0) * nk,
        "launches_per_step": dom.get("launches_per_step"), "avg_launch_ms": dom.get("avg_launch_ms"),
        "kernel_share_of_step": dom.get("share_of_step"),
        "note": ("one 8-bit digit pass over 64-bit suffix records (read once, written once); the build runs 4 of them. "
                 "build.frac compares the whole build with SURVEY 8(d)'s prefix-doubling byte model: the "
                 "uniform read-set path replaces the model's doubling rounds by one verified overlap per read, so the "
                 "build moves ~130 B/suffix and that fraction exceeds 1"),
        "build": {"alg_bytes_per_suffix": per_suffix, "P": P, "R16": R16,
                  "achieved_gbs": per_suffix * n / (ms_per_step * 1e-3) / 1e9,
                  "frac": per_suffix * n / (ms_per_step * 1e-3) / 1e9 / peak},
        "kernels": kernels,
        "sum_kernel_ms_per_step": kernel_ms,
    }


def cpu_sa_baseline(text: np.ndarray, L: int) -> dict:
    """The reference's build_parallel (all host threads) on a bounded prefix of `text`, plus its other
    two routes to the same array on one thread."""
    cpu_lib, kind = _load_cpu_lib()
    cores = os.cpu_count() or 1
    workers = cores if kind == "reference" else 1
    probe = cpu_sample(text, L, 1 << 17)
    t_probe = cpu_build(cpu_lib, kind, probe, workers)
    sample = cpu_sample(text, L, int(min(1 << 22, max(1 << 17, probe.size * (15.0 / t_probe) ** (1 / 1.35)))))
    dt = cpu_build(cpu_lib, kind, sample, workers)
    also = None
    if kind == "reference":   # the reference's other two ways to the same array, one thread each
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        tmp = np.empty(sample.size, np.uint32)
        t0 = time.perf_counter()
        cpu_lib.ref_build_naive(vp(sample), C.c_size_t(sample.size), vp(tmp), None)
        t_naive = time.perf_counter() - t0
        small = cpu_sample(text, L, 1 << 17)
        t_one = cpu_build(cpu_lib, kind, small, 1)
        also = {"build_naive_1_thread_msuffixes_per_s": sample.size / t_naive / 1e6,
                "build_parallel_1_worker_msuffixes_per_s": small.size / t_one / 1e6,
                "build_parallel_1_worker_sample_suffixes": int(small.size)}
    return {"value": sample.size / dt / 1e6, "unit": UNIT, "cores": workers, "kind": kind, "also": also,
            "sample": f"first {sample.size // (L + 1)} reads ({sample.size} suffixes) of the same text, 1 build, "
                      f"{dt:.1f} s; reference build_parallel with executor{{workers={workers}}}" if kind == "reference"
            else f"first {sample.size} suffixes, oracle port, 1 thread, {dt:.1f} s"}


def ncu_overlap_traffic(workload: str) -> dict:
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the overlap kernels, from the ncu
    --set full captures committed under profiles/ (r2_ncu_overlap_traffic.json: {workload: {kernel: bytes}})."""
    p = ROOT / "profiles" / "r2_ncu_overlap_traffic.json"
    if p.exists():
        try:
            return {k: float(v) for k, v in json.loads(p.read_text()).get(workload, {}).items()}
        except Exception:
            pass
    return {}


def cpu_query_baseline(G: int, L: int, k: int, min_overlap: int = 20) -> dict:
    """The overlap job's query stream through the reference's own fragment_index::locate_prefix_range
    (fragment_index.hpp:65-70) on this box's host cores: 1 thread and all threads over one shared index
    of a labelled prefix of the reads, a bounded number of queries each."""
    lib, kind = _load_cpu_lib()
    if kind != "reference":
        return {"unavailable": "oracle/_ref not present: the reference's fragment_index cannot be timed"}
    kk = min(k, (1 << 21) // (L + 1))
    text = cpu_read_text(G, L, kk)
    starts = (np.arange(kk, dtype=np.uint32) * np.uint32(L + 1))
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    lib.ref_index_create_from_text.restype = C.c_void_p
    lib.ref_index_query_bench.restype = C.c_double
    t0 = time.perf_counter()
    h = lib.ref_index_create_from_text(vp(text), C.c_size_t(text.size), vp(starts), C.c_size_t(kk), 0, 0, 1, C.c_size_t(1 << 15))
    t_build = time.perf_counter() - t0
    if not h:
        return {"unavailable": "reference index construction failed"}
    cores = os.cpu_count() or 1
    out = {"kind": "reference", "unit": "Mqueries/s", "what": "fragment_index::locate_prefix_range (fragment_index.hpp:65-70)",
           "sample": f"index (builder::direct, {t_build:.1f} s) over the first {kk} reads ({text.size} suffixes) of the same text; "
                     f"query stream = every read suffix of length >= {min_overlap}"}
    for label, threads, budget in (("1_thread", 1, 400_000), ("all_threads", cores, 400_000 * min(cores, 16))):
        done, acc = C.c_uint64(0), C.c_uint64(0)
        sec = lib.ref_index_query_bench(C.c_void_p(h), C.c_uint32(min_overlap), C.c_uint(threads), C.c_uint64(budget), 0,
                                        C.byref(done), C.byref(acc))
        out[label] = {"value": done.value / sec / 1e6, "threads": threads, "queries": int(done.value), "seconds": sec}
    done, acc = C.c_uint64(0), C.c_uint64(0)
    sec = lib.ref_index_query_bench(C.c_void_p(h), C.c_uint32(min_overlap), C.c_uint(cores), C.c_uint64(100_000 * min(cores, 16)), 1,
                                    C.byref(done), C.byref(acc))
    out["prefix_related_all_threads"] = {"value": done.value / sec / 1e6, "threads": cores, "queries": int(done.value),
                                         "seconds": sec, "what": "fragment_index::prefix_related (fragment_index.hpp:72-109)"}
    out["value"] = out["all_threads"]["value"]
    out["cores"] = cores
    lib.ref_index_destroy(C.c_void_p(h))
    return out


# ---- main arm ----------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--no-overlap", action="store_true", help="skip the overlap-query measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines")
    ap.add_argument("--no-routes", action="store_true", help="skip the general-route measurements")
    ap.add_argument("--sweep", action="store_true",
                    help="SA build throughput over n = 2^20, 2^22, ... full (BASELINE config 3's sweep; implied by --workload c3)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-GPU code path (sharded.bench_main) even with one rank: a plumbing check")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    workload = args.workload or "c2"
    G, L, k = WORKLOADS[workload]

    if args.impl == "reference":
        if rank != 0:
            return
        # the arm maps oracle/ only (never the product library): the text generator is the reference's
        # own make_fragment_set over its own RNG draws (oracle/ref_shim.cpp ref_make_read_text), or the
        # oracle port's restatement of it.  A prefix of the reads is all the arm needs (2^22 bytes' worth).
        kk = min(k, (1 << 22) // (L + 1) + 1)
        run_reference(args, cpu_read_text(G, L, kk), L, workload)
        return

    import torch
    import torch.distributed as dist
    import paper_1404_3456_b200 as rq

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the reseq B200 backend has no CPU fallback")
    torch.cuda.set_device(local_rank)
    if world > 1 or args.force_sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        os.environ.setdefault("NCCL_DEBUG", "WARN")   # (NCCL's version banner would otherwise precede the JSON line on stdout)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        # (the default workload stays config 2 for every N so that the driver's per-N values are comparable;
        #  --workload c4 / c5 are the configurations the sharded build is meant for)

    if world > 1 or args.force_sharded:
        from paper_1404_3456_b200 import sharded
        sharded.bench_main(args, workload, rank, world, local_rank)
        return

    # ---- inputs: RNG-exact synthetic read text, pinned on the host, resident in HBM -----------
    text, starts = rq.synth_read_text(G, L, k, 1, 2, pinned=True)
    n = int(text.size)
    ex = rq.Executor(local_rank)
    # everything below runs on ONE explicit stream: the library launches on it, torch allocates and
    # copies on it, and the timing events are recorded on it (CUDA events see only their own stream)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ex.set_stream(stream.cuda_stream)
    lib = rq._lib.load()
    d_text = torch.from_numpy(text).cuda()
    d_sa = torch.empty(n, dtype=torch.int32, device="cuda")
    d_rank = torch.empty(n, dtype=torch.int32, device="cuda")
    st = rq.SaStats()

    def step_device():
        rq._lib.check(lib.reseq_cuda_build_sa_device(ex.handle, C.c_void_p(d_text.data_ptr()), n,
                                                     C.c_void_p(d_sa.data_ptr()), C.c_void_p(d_rank.data_ptr()),
                                                     C.byref(st)))

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    # Timed region: K builds as a caller runs them (no per-launch events: a repeated device-resident build is
    # replayed as one CUDA graph).  The per-kernel table behind `roofline` comes from K further builds of the same
    # loop, right after, with CUDA events around every launch (those builds launch kernel by kernel and are
    # reported as ms_per_step_with_launch_events).
    launches0 = ex.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step_device()
        ev1.record(stream)
        torch.cuda.synchronize()
        ms_total = ev0.elapsed_time(ev1)
        launches = ex.launch_count - launches0
        ex.profile(True)
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(args.steps):
            step_device()
        ev3.record(stream)
        torch.cuda.synchronize()
        ms_profiled = ev2.elapsed_time(ev3) / args.steps
        prof = ex.profile_read()
        ex.profile(False)
    ms_per_step = ms_total / args.steps
    value = n / (ms_per_step * 1e-3) / 1e6

    # parity fingerprint of what was just built (size-independent proof runs in tests/)
    sa_host = d_sa.cpu().numpy().view(np.uint32)
    # rank[sa[i]] == i for every i  <=>  sa is a permutation and rank its inverse
    perm_ok = True
    chunk = 1 << 28   # in pieces: the int64 index tensors of 3 G suffixes would not fit next to the build's arena
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        pos = d_sa[lo:hi].to(torch.int64) & 0xFFFFFFFF
        back = d_rank[pos].to(torch.int64) & 0xFFFFFFFF
        perm_ok = perm_ok and bool(torch.equal(back, torch.arange(lo, hi, device="cuda", dtype=torch.int64)))
        del pos, back

    # ---- roofline: per-kernel algorithmic bytes over live CUDA-event durations ----
    peak, peak_src = measured_peak()
    per_suffix, P, R16 = bytes_alg_per_suffix(n, L)
    roofline = roofline_block(prof, n, L, args.steps, ms_per_step, workload)

    # ---- e2e: host buffers through the C ABI -----------------------------------------------------
    h_sa = torch.empty(n, dtype=torch.int32).pin_memory()
    h_rank = torch.empty(n, dtype=torch.int32).pin_memory()

    def step_host():
        rq._lib.check(lib.reseq_cuda_build_sa(ex.handle, C.c_void_p(text.ctypes.data), n,
                                              C.c_void_p(h_sa.data_ptr()), C.c_void_p(h_rank.data_ptr()), None))

    step_host()
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    same = bool(np.array_equal(h_sa.numpy().view(np.uint32), sa_host))
    e2e = {"value": n / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": n, "d2h_bytes_per_step": 8 * n,
           "ms_per_step": e2e_s * 1e3, "steps": e2e_steps, "matches_device_run": same}

    peak_frac = lambda b, ms: b / (ms * 1e-3) / 1e9 / peak

    def timed_builds(executor, dn_text, dn, steps, warm=1):
        """ms per device-resident build of the first dn bytes of the text on `executor`."""
        s2 = rq.SaStats()
        run = lambda: rq._lib.check(lib.reseq_cuda_build_sa_device(executor.handle, C.c_void_p(dn_text.data_ptr()), dn,
                                                                    C.c_void_p(d_sa.data_ptr()), C.c_void_p(d_rank.data_ptr()),
                                                                    C.byref(s2)))
        for _ in range(warm):
            run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(steps):
            run()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps, s2

    # ---- the general routes on the same text (what ragged reads / other alphabets take) -----------
    routes = None
    if not args.no_routes and n <= 400_000_000:
        routes = {}
        for name, opt in (("general_dna", ("sa_uniform", 0)), ("doubling", ("sa_text_rounds", 0))):
            e2 = rq.Executor(local_rank)
            e2.set_stream(stream.cuda_stream)
            e2.set_option(*opt)
            ms_r, st_r = timed_builds(e2, d_text, n, 3)
            e2.close()
            routes[name] = {"option": f"{opt[0]}={opt[1]}", "ms_per_build": ms_r, "msuffixes_per_s": n / (ms_r * 1e-3) / 1e6,
                            "vs_default_route": ms_r / ms_per_step, "rounds": int(st_r.rounds),
                            "sort_passes": int(st_r.sort_passes), "init_symbols": int(st_r.init_symbols),
                            "frac_of_8d_model": peak_frac(per_suffix * n, ms_r)}

        # a ragged read set of the same genome and read count (lengths 100 .. L: trimmed reads), default options
        if G >= 2 * L:
            rng = np.random.default_rng(7)
            genome = rq.synth_random_dna(G, 1)
            lens = rng.integers(max(16, L - 50), L + 1, k)
            st0 = rng.integers(0, G - L, k)
            total = int(lens.sum()) + k
            offs = np.concatenate(([0], np.cumsum(lens + 1)[:-1]))
            idx = np.minimum(np.repeat(st0 - offs, lens + 1) + np.arange(total), G - 1)
            rag = genome[idx]
            rag[offs + lens] = 0
            del idx
            d_rag = torch.from_numpy(rag).cuda()
            e2 = rq.Executor(local_rank)
            e2.set_stream(stream.cuda_stream)
            ms_r, st_r = timed_builds(e2, d_rag, total, 3)
            e2.close()
            b_r, _, _ = bytes_alg_per_suffix(total, L)
            routes["ragged_reads"] = {"option": f"default options; read lengths uniform in {max(16, L - 50)}..{L}", "suffixes": total,
                                      "ms_per_build": ms_r, "msuffixes_per_s": total / (ms_r * 1e-3) / 1e6,
                                      "vs_default_route_per_suffix": (ms_r / total) / (ms_per_step / n), "rounds": int(st_r.rounds),
                                      "sort_passes": int(st_r.sort_passes), "init_symbols": int(st_r.init_symbols),
                                      "frac_of_8d_model": peak_frac(b_r * total, ms_r)}
            del d_rag, rag

    # ---- BASELINE config 3: throughput sweep over n by truncating k ---------------------------------
    sweep = None
    if args.sweep or workload == "c3":
        sweep = []
        sizes = [e for e in range(20, 40, 2) if (1 << e) < n]
        for kk in [max(1, (1 << e) // (L + 1)) for e in sizes] + [k]:
            dn = kk * (L + 1)
            ms_s, _ = timed_builds(ex, d_text, dn, 10 if dn < (1 << 26) else 5, warm=2)
            b_s, _, _ = bytes_alg_per_suffix(dn, L)
            sweep.append({"reads": kk, "suffixes": dn, "ms_per_build": ms_s, "msuffixes_per_s": dn / (ms_s * 1e-3) / 1e6,
                          "frac_of_8d_model": peak_frac(b_s * dn, ms_s)})

    # ---- overlap queries -------------------------------------------------------------------------
    overlap = None
    if not args.no_overlap:
        del h_rank
        fset = rq.fragment_set_from_text(text, starts)
        rq.FragmentIndex(fset, ex).close()    # warm-up: arena growth, pool allocations
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix = rq.FragmentIndex(fset, ex)
        torch.cuda.synchronize()
        t_index = time.perf_counter() - t0
        # per-kernel table of one more index build (CUDA events around every launch add their own cost:
        # this build is not the one timed above)
        ex.profile(True)
        rq.FragmentIndex(fset, ex).close()
        ix_prof = ex.profile_read()
        ex.profile(False)
        index_kernels = {kname: {"ms": ms, "launches": cnt} for kname, (cnt, ms) in sorted(ix_prof.items(), key=lambda kv: -kv[1][1])}
        ix.overlaps(20, reuse_buffers=True)  # warm-up (arena growth, page-locked result arrays)
        ex.profile(True)
        t0 = time.perf_counter()
        ov = ix.overlaps(20, reuse_buffers=True)
        t_ov = time.perf_counter() - t0
        ov_prof = ex.profile_read()
        ex.profile(False)
        q_alg = 2 * int(np.ceil(np.log2(n))) * 64 + 64
        traffic = ncu_overlap_traffic(workload)
        ov_kernels = {}
        for kname, (cnt, ms) in sorted(ov_prof.items(), key=lambda kv: -kv[1][1]):
            tr = traffic.get(kname)
            ov_kernels[kname] = {"ms": ms, "launches": cnt, "share": ms / ov.device_ms if ov.device_ms else None,
                                 "dram_bytes_ncu": tr, "dram_gbs": tr / (ms * 1e-3) / 1e9 if tr and ms else None,
                                 "dram_frac_of_peak": tr / (ms * 1e-3) / 1e9 / peak if tr and ms else None}
        dom_ov = next(iter(ov_kernels)) if ov_kernels else None
        dom_rec = ov_kernels.get(dom_ov, {})
        overlap = {"metric": "overlap_queries_per_s", "min_overlap": 20, "queries": ov.queries,
                   "value": ov.queries / (ov.device_ms * 1e-3) / 1e6, "unit": "Mqueries/s",
                   "device_ms": ov.device_ms,
                   "e2e": {"value": ov.queries / t_ov / 1e6, "unit": "Mqueries/s", "ms": t_ov * 1e3,
                           "h2d_bytes": 8 * (k + 1), "d2h_bytes": int(12 * ov.i.size + k),
                           "note": "index resident; query offsets in, (i, j, w) triples + containment flags out to page-locked host arrays"},
                   "overlaps_found": int(ov.i.size),
                   "contained_reads": int(ov.contained.sum()), "index_build_ms": t_index * 1e3,
                   "index_build_kernels": index_kernels, "index_build_kernel_ms": sum(v["ms"] for v in index_kernels.values()),
                   "roofline": {"bound": "hbm", "kernel": dom_ov, "peak": peak, "unit": "GB/s",
                                "traffic": dom_rec.get("dram_bytes_ncu"), "achieved": dom_rec.get("dram_gbs"),
                                "frac": dom_rec.get("dram_frac_of_peak"),
                                "alg_bytes_per_query_cold_model": q_alg,
                                "cold_model_frac": q_alg * ov.queries / (ov.device_ms * 1e-3) / 1e9 / peak,
                                "note": ("achieved = ncu dram bytes of the dominant kernel / its CUDA-event time in this run. "
                                         "SURVEY 8(d)'s cold binary-search model (2 ceil(log2 n) x 64 + 64 B/query) assumes ~2 log n "
                                         "DRAM probes; the directory + rank anchor need ~1 DRAM gather per query, so the cold-model "
                                         "fraction is above 1 and is reported only for continuity"),
                                "kernels": ov_kernels}}
        ix.close()
        if not args.no_cpu:
            overlap["cpu_baseline"] = cpu_query_baseline(G, L, k)

    # ---- CPU baseline -------------------------------------------------------------------------------
    cpu = None if args.no_cpu else cpu_sa_baseline(text, L)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "ms_per_step_with_launch_events": ms_profiled,
        "kernel_timing": "timed region = K builds without per-launch events (a repeated device-resident build replays as one "
                         "CUDA graph); roofline.kernels = CUDA events around every launch of K further builds run right after",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": {"workload": DESCRIPTION[workload], "genome_bp": G, "read_len": L, "reads": k, "suffixes": n,
                   "l2_policy": (f"inputs larger than L2 (text {n / 1e6:.0f} MB, record arrays {8 * n / 1e6:.0f} MB each, "
                                 f"sa / rank {4 * n / 1e6:.0f} MB each vs 126 MB L2)")
                   if 4 * n > 256_000_000 else "working set exceeds L2 only partly; no flush",
                   "rounds": int(st.rounds), "init_symbols": int(st.init_symbols),
                   "sort_passes": int(st.sort_passes), "alphabet": "dna-2bit" if st.alphabet == 0 else "bytes"},
        "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": int(launches),
        "roofline": roofline, "cpu_baseline": cpu, "overlap": overlap, "routes": routes, "sweep": sweep,
        "checks": {"rank_is_inverse_of_sa": perm_ok, "host_run_equals_device_run": same},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
