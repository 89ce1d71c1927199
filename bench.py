#!/usr/bin/env python
"""Benchmark of the TACOS-Greedy hot path on B200 (BASELINE.json metric:
"link-chunk matches/sec and 512-NPU All-Reduce synthesis wall time").

One step = one best-of-S All-Reduce synthesis of the workload (config 3 by
default: 3-D torus 8x8x8, 512 NPUs, 1 chunk/NPU of 1 MiB, 64 seeds per GPU):
the batched greedy search (rows a2-a6), best-of-S selection (a7; across GPUs
one NCCL MIN all-reduce of two uint64 keys) and the winner's emission with the
RS inversion and AR composition (a8).  Inputs (topology, plan state) are
resident in HBM when the timed region starts; L2 is flushed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--config 3] [--impl reference]

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
(oracle/, plain C, the parity reference) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "link-chunk matches/sec and 512-NPU All-Reduce synthesis wall time"
UNIT = "matches/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seeds", type=int, default=0, help="seeds per GPU (default: the config's)")
    ap.add_argument("--impl", default="tacos", choices=["tacos", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="steps of the end-to-end leg (default = steps)")
    ap.add_argument("--literal", action="store_true", help="paper-literal chunk-first variant (row f1)")
    ap.add_argument("--no-baselines", action="store_true", help="skip the continuous-time Ring/Direct comparison")
    return ap.parse_args()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def usable_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def workload(cfg: int, seeds: int):
    wl = W.config(cfg)
    if seeds:
        wl.n_seeds = seeds
    return wl


def matches_per_seed(wl) -> int:
    n = wl.topo.n_npus
    return n * wl.chunks_per_npu * (n - 1)


# --------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------
def oracle_sample(wl, budget_s: float = 0.0, seeds_cap: int = 0):
    """Time the oracle, as it stands, on a bounded sample of the workload (about 20 s of CPU
    work): seeds run one per host thread (the oracle is single-threaded per seed)."""
    import oracle

    cores = usable_cores()
    budget_s = budget_s or max(1.0, 20.0 / cores)  # wall seconds
    t0 = time.perf_counter()
    g1 = oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, "AG", [0], record=False)
    one = time.perf_counter() - t0
    if one > budget_s:  # one seed already exceeds the budget (config 4): that seed is the sample
        m = sum(g.M for g in g1.ag)
        return {"value": m / one, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"{wl.name}: 1 of {wl.n_seeds} seeds, the AG search of seed 0 without emission "
                          f"(one seed alone takes {one:.1f} s), 1 thread ({cpu_model()})",
                "seconds": one, "seeds": 1}
    per_thread = max(1, int(budget_s / max(one, 1e-3)))
    n = min(cores * per_thread, wl.n_seeds if not seeds_cap else seeds_cap)
    n = max(1, n)
    seeds = list(range(n))
    # the sample: the workload's best-of-n synthesis, repeated (with the next seeds) until about
    # budget_s of wall time has been spent, so a fast oracle run is still measured over seconds
    dt, m, rounds = 0.0, 0, 0
    while rounds == 0 or dt < budget_s:
        base = rounds * n
        t0 = time.perf_counter()
        syn = oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, wl.collective,
                                [base + s for s in seeds], threads=cores)
        dt += time.perf_counter() - t0
        m += sum(g.M for g in syn.ag) + (sum(g.M for g in syn.rs) if syn.rs is not syn.ag else 0)
        rounds += 1
        del syn
    return {"value": m / dt, "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
            "sample": f"{wl.name}: {rounds} x best-of-{n} {wl.collective} syntheses (seeds 0..{rounds * n - 1}; the "
                      f"workload has {wl.n_seeds} seeds) incl. emission, {dt:.2f} s wall on {min(cores, n)} threads "
                      f"({cpu_model()})",
            "seconds": dt, "seeds": n * rounds}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args.config, args.seeds)
    cores = usable_cores()
    import oracle

    # one step = `cores` seeds (one per thread) of the workload, the oracle as it stands
    seeds_per_step = min(cores, wl.n_seeds)
    times = []
    m_step = 0
    for i in range(args.warmup + args.steps):
        seeds = [(i * seeds_per_step + s) % (2**64) for s in range(seeds_per_step)]
        t0 = time.perf_counter()
        syn = oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, wl.collective, seeds, threads=cores)
        dt = time.perf_counter() - t0
        m_step = sum(g.M for g in syn.ag) + (sum(g.M for g in syn.rs) if syn.rs is not syn.ag else 0)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = m_step * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": wl.name, "npus": wl.topo.n_npus, "links": wl.topo.n_links,
                   "chunks_per_npu": wl.chunks_per_npu, "chunk_bytes": wl.chunk_bytes, "collective": wl.collective,
                   "seeds_per_step": seeds_per_step, "note": "CPU oracle (plain C, single-threaded per seed)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": seeds_per_step, "kind": "oracle",
                         "sample": f"{seeds_per_step} seeds of {wl.name} per step on {seeds_per_step} threads ({cpu_model()})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# clocks sampling during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.proc = None
        self.lines = []
        self.thr = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thr = threading.Thread(target=self._read, daemon=True)
        self.thr.start()
        t_end = time.time() + 5.0  # nvidia-smi start-up (slow with several ranks): wait for the first sample
        while not self.lines and time.time() < t_end and self.proc.poll() is None:
            time.sleep(0.01)
        self.lines.clear()  # keep only the samples taken from here on (the timed region)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thr:
            self.thr.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def algorithmic_bytes(stats: dict, n_chunks: int) -> int:
    """B = V (R + 16) + D (2R) + 48 M, R = C/8 bytes per row."""
    R = n_chunks / 8.0
    return int(stats["visits"] * (R + 16) + stats["dest_events"] * 2 * R + 48 * stats["matches"])


def touched_bytes(stats: dict, n_chunks: int) -> int:
    """What the kernels move given the exact skip: a live visit reads the source row and the
    destination's have row (2R) plus 16 B of link state, a skipped visit (source unchanged since
    the link's last empty visit: provably no candidate) only the 16 B, a match 48 B (record +
    arrival): Lv (2R + 16) + (V - Lv) 16 + 48 M, Lv = live visits counted by the kernels."""
    R = n_chunks / 8.0
    lv = stats.get("live_visits", stats["visits"])
    return int(lv * (2 * R + 16) + (stats["visits"] - lv) * 16 + 48 * stats["matches"])


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2304_05301_b200 as T

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    T.load_library()
    comm = None
    if world > 1:
        # the exchange step of best-of-S runs inside the library (tacos_plan_allreduce_keys:
        # ncclAllReduce MIN over NVLink); torch.distributed only ships the NCCL id, the barriers
        # and the max-over-ranks timing
        obj = [T.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = T.Comm(obj[0], world, rank)
    wl = workload(args.config, args.seeds)
    S = wl.n_seeds
    C = wl.topo.n_npus * wl.chunks_per_npu
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    topo = T.Topology.from_workload_topology(wl.topo)
    plan = T.Plan(topo, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S, 0, rank * S, literal=args.literal)
    n_sends = plan.n_sends
    d_sends = torch.empty(n_sends * 32, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(ev):
        # search -> (key all-reduce) -> emission queued back to back; the winner is resolved on
        # the device where the plan allows it, and the host reads the result after the step
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            plan.search(sh)
            ev[1].record(stream)
            if world > 1:
                plan.allreduce_keys(comm, sh)
            if plan.emit_async(d_sends.data_ptr(), n_sends, sh):
                ev[2].record(stream)
                res = plan.result(n_sends, sh)
            else:
                res = plan.emit(d_sends.data_ptr(), n_sends, sh)
                ev[2].record(stream)
        return res

    launches_per_step = None
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
        launches_per_step = plan.last_launches()
    stats = plan.stats(sh)
    clocks = ClockSampler(dev)
    clocks.start()
    barrier()
    evs = []
    res = None
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush, outside the timed events
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        res = step(ev)
        evs.append(ev)
        launches_per_step = plan.last_launches() + 2  # emit launches + search launches (greedy, best_keys)
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(c) for a, b, c in evs]
    search_ms = [a.elapsed_time(b) for a, b, c in evs]
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms, sum(search_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, tot_search_ms = float(t[0]), float(t[1])
    m_step_local = stats["matches"]
    m_total = m_step_local * world  # weak scaling: every rank searches its own S seeds
    value = m_total * args.steps / (tot_ms / 1e3)
    # roofline of the dominant kernel (greedy search): algorithmic bytes / kernel time, against
    # the memory level that serves them: shared memory when the plan keeps the
    # per-seed bitsets on chip (configs 1-3, 5), else HBM (config 4; L2-resident below 126 MB)
    # achieved = the bytes the kernels move per launch given the exact skip; SURVEY
    # §8(d)'s B (a row per visit, two per destination-event) is reported beside it
    B_survey = algorithmic_bytes(stats, C)
    B = touched_bytes(stats, C)
    search_avg_s = sum(search_ms) / len(search_ms) / 1e3
    achieved = B / search_avg_s / 1e9
    survey_gbs = B_survey / search_avg_s / 1e9
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    info = plan.info()
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    smem_peak = n_sms * 128 * sm_mhz * 1e6 / 1e9  # 128 B/clk/SM shared-memory crossbar (B300_MICROARCH.md)
    ncu = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            data = json.load(fh)
            ncu = data.get(f"{wl.name}_s{S}") or (data.get(wl.name) if S == W.config(args.config).n_seeds else None) or {}
    except (OSError, ValueError):
        pass
    traffic = ncu.get("dram_bytes_per_launch")
    if info["rows_in_smem"]:
        bound, peak = "smem", smem_peak
        peak_src = f"derived: {n_sms} SMs x 128 B/clk x {sm_mhz:.0f} MHz (shared-memory crossbar, B300_MICROARCH.md)"
    else:
        bound, peak, peak_src = "hbm", hbm_peak, hbm_src
    roofline = {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": "greedy_kernel (+best_keys)", "peak_source": peak_src,
        "algorithmic_bytes_per_launch": B,
        "bytes_definition": "Lv (2R+16) + (V-Lv) 16 + 48 M, R = C/8: a live visit reads the source row and the "
                            "destination's have row, a visit skipped exactly (source unchanged) 16 B of link state, "
                            "a match 48 B; Lv = live visits counted by the kernels",
        "survey_bytes_per_launch": B_survey,
        "frac_survey_bytes": survey_gbs / peak,
        "frac_vs_hbm": achieved / hbm_peak,
        "dram_frac_of_hbm": (traffic / search_avg_s / 1e9 / hbm_peak) if traffic else None,
        "smem_pipe_frac": ncu.get("smem_pipe_frac"), "issue_active_pct": ncu.get("issue_active_pct"),
        "warps_active_pct": ncu.get("warps_active_pct"), "ncu_source": ncu.get("source"),
        "grid": {"ctas": info["ctas"], "sms": n_sms, "cluster": info["cluster"], "threads": info["threads"],
                 "smem_bytes": info["smem_bytes"], "rows_bytes_global": info["rows_bytes"],
                 "event_loop": {0: "per-event", 1: "windowed", 2: "lock-step"}.get(info.get("event_loop"), "?")},
        "limiter": ("latency: per-event dependent walks of each destination and "
                    + ("one cluster barrier per event (lock-step loop" if info.get("event_loop") == 2
                       else "two cluster barriers per event (per-event loop")
                    + ", DESIGN.md §5); neither HBM nor the shared-memory pipe is saturated") if info["rows_in_smem"] else
                   ("latency: L2 round trips of the 1 KiB source rows in the windowed loop and three cluster barriers "
                    "per window (DESIGN.md §5); rows are " + ("L2-resident" if info["rows_bytes"] < 126e6 else
                                                              "larger than L2") + ", DRAM traffic is the send records"),
    }

    # ---- e2e: public C-ABI call with host buffers (topology upload + synth + D2H) ----
    e2e_steps = args.e2e_steps or args.steps
    host_out = torch.empty(n_sends * 32, dtype=torch.uint8).pin_memory()
    src_h = np.ascontiguousarray(wl.topo.src)
    h2d = wl.topo.n_links * 16
    d2h = 0
    e2e_ms = []
    p_e2e, keep = T.make_params(wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S, 0, rank * S,
                                flags=T.TACOS_FLAG_LITERAL if args.literal else 0)
    for i in range(1 + e2e_steps):
        barrier()
        t0 = time.perf_counter()
        tt = T.Topology(wl.topo.n_npus, src_h, wl.topo.dst, wl.topo.alpha_ns, wl.topo.bw)
        if world == 1:
            r = T.synthesize_into(tt, p_e2e, host_out.data_ptr(), n_sends, sh)
            d2h = n_sends * 32
        else:
            pl = T.Plan(tt, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S, 0, rank * S)
            with torch.cuda.stream(stream):
                pl.search(sh)
                pl.allreduce_keys(comm, sh)
                r = pl.emit(d_sends.data_ptr(), n_sends, sh)
                if r["winner_local"]:
                    host_out.copy_(d_sends, non_blocking=True)
            stream.synchronize()
            d2h = n_sends * 32 if r["winner_local"] else 0
            del pl
        del tt
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_ms.append(dt * 1e3)
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = m_total * len(e2e_ms) / (float(e2e_t[0]) / 1e3)

    # continuous-time collective time of the winning schedule vs the Ring / Direct
    # baselines (row f3): the paper's normalized comparison
    coll_times = None
    if rank == 0 and not args.no_baselines and world == 1:
        sends_h = T.sends_from_bytes(host_out.numpy())
        tac = T.evaluate_continuous(topo, sends_h, wl.collective, wl.chunks_per_npu, wl.chunk_bytes)["T_ns"]
        coll_times = {"tacos_us": tac / 1e3}
        n = wl.topo.n_npus
        for alg in ("ring", "direct"):
            est = n * (n - 1) * wl.chunks_per_npu * (8 if alg == "direct" else 2)
            if est > 40_000_000:  # the baseline schedule alone would need several GB of host memory
                coll_times[alg + "_us"] = None
                continue
            bs = T.baseline(topo, alg, wl.collective, wl.chunks_per_npu, wl.chunk_bytes)
            coll_times[alg + "_us"] = T.evaluate_continuous(topo, bs, wl.collective, wl.chunks_per_npu,
                                                            wl.chunk_bytes)["T_ns"] / 1e3
            coll_times["speedup_vs_" + alg] = coll_times[alg + "_us"] / coll_times["tacos_us"]

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_sample(wl)
            cpu.pop("seconds", None)
            cpu.pop("seeds", None)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl.name, "npus": wl.topo.n_npus, "links": wl.topo.n_links,
                       "chunks_per_npu": wl.chunks_per_npu, "chunk_bytes": wl.chunk_bytes,
                       "collective": wl.collective, "seeds_per_gpu": S, "seeds_total": S * world,
                       "parallelism": f"seed-sharded x{world}", "l2": "flushed between steps (256 MiB write)"},
            "synthesis_ms": statistics.median(step_ms), "synthesis_ms_first": step_ms[0],
            "search_ms": tot_search_ms / args.steps, "T_ar": res["T"], "T_ag": res["T_ag"], "T_rs": res["T_rs"],
            "winner_seed": res["seed"], "matches_per_step": m_total, "n_sends": n_sends,
            "paper_context": "TACOS-Greedy 512-NPU AR synthesis 6.09 min (P:L354, Ring_FC_Switch, hardware not stated)",
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": float(e2e_t[0]) / len(e2e_ms)},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"],
                       "samples": clk["samples"]},
            "stats": {"V": stats["visits"], "D": stats["dest_events"], "M": stats["matches"], "E": stats["events"],
                      "Lv": stats.get("live_visits"), "cancelled": stats.get("cancelled", 0)},
            "variant": "paper-literal chunk-first + replacement (f1)" if args.literal else "link-first (R1, R4)",
            "collective_time": coll_times,
            "wall_s": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
