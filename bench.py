#!/usr/bin/env python
"""bench.py -- triangle-count GTEPS (|E|/time) on B200, BASELINE.json's metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference        # the reference's own CPU path

Workload (config.workload): RMAT scale-24 edgefactor-16 with per-vertex
counts (BASELINE.json configs[3], the configuration the metric's "1/2/4/8
B200" is quoted on; it fits one GPU).  Synthetic, deterministic (SURVEY.md 8d
splitmix generator, generated on the device).

A step = one triangle count of the whole graph from the resident oriented CSR:
level-1 frontier + degree-binned advance/join + reduce (total and per-vertex),
plus at N>1 the NCCL allreduce of the per-rank partial counts.  `value` =
|E| / step time (GTEPS, whole job).  `e2e` = the same through the
reference-facing drop-in call count_triangles(const Graph&) with HOST buffers:
H2D of the symmetric CSR (pinned) + orientation + count + D2H of the total and
per-vertex array, every step.
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

CONFIGS = {
    # name: (kind, scale, param, per_vertex, description)
    "C1": ("rmat", 16, 16, False, "RMAT scale-16 edgefactor-16 (configs[0])"),
    "C2": ("er", 20, 32, False, "Erdos-Renyi G(n=2^20, avg degree 32) (configs[1])"),
    "C3": ("kron", 22, 16, False, "Graph500 Kronecker scale-22 edgefactor-16, permuted (configs[2])"),
    "C4": ("rmat", 24, 16, True, "RMAT scale-24 edgefactor-16 with per-vertex counts (configs[3])"),
    "C5": ("rmat", 26, 32, False, "RMAT scale-26 edgefactor-32, total count (configs[4])"),
}
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--no-per-vertex", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of CUDA-graph replay")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.n_during = len(self.lines)
        if self.proc and not self.lines:
            # a timed region shorter than nvidia-smi's start-up: take the first
            # sample right after it (flagged in the summary)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3 and self.proc.poll() is None:
                time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "n_during", 1) == 0:
            out["sampled"] = "right after the timed region (shorter than nvidia-smi start-up)"
        return out


def gen_kind(tc, kind):
    return {"rmat": tc.GEN_RMAT, "kron": tc.GEN_KRON, "er": tc.GEN_ER}[kind]


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own count_triangles path (oracle/_ref, built
# from /root/reference's sources) on a bounded, cost-stratified seed sample,
# extrapolated by the reference's per-row visit cost model.
# ---------------------------------------------------------------------------
_CAL = None


def calibration():
    """Ratio (full trimatch::count_triangles time) / (sample estimate) on C1,
    the one config where the reference's full run takes seconds."""
    global _CAL
    if _CAL is None:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle_ctypes import Oracle, Ref
        o = Oracle()
        off, nb, E, _, _ = o.build_graph(o.gen_rmat(16, 16), 1 << 16)
        rg = Ref().graph(off, nb)
        t0 = time.perf_counter()
        T = rg.count_triangles(lookahead=2, workers=0)
        full_ms = (time.perf_counter() - t0) * 1e3
        est = reference_cpu_sample(off, nb, 2.0, E, rg, calibrate=False)
        _CAL = {"config": "C1 RMAT s16 ef16", "full_ms": full_ms, "sample_est_ms": est["t_sample_est_ms"],
                "factor": full_ms / est["t_sample_est_ms"], "triangles": T}
    return _CAL


def reference_cpu_sample(off: np.ndarray, nb: np.ndarray, budget_s: float, E: int, rg=None, calibrate=True):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_ctypes import REF_SO, Oracle, Ref
    if not os.path.exists(REF_SO):
        return None
    ref = Ref()
    t_wall0 = time.perf_counter()
    if rg is None:
        rg = ref.graph(off, nb)
    # visits the final level makes for seed u: deg(u) per level-1 row (u,w),
    # w in N(u), w > u (matcher.cpp:215-228); cost-stratified systematic sample
    cost = Oracle().seed_costs(off, nb)
    total_cost = float(cost.sum())
    order = np.argsort(cost, kind="stable")[::-1]
    order = order[cost[order] > 0]
    workers = os.cpu_count() or 1
    # seeds: a cost-stratified systematic sample (~2048 seeds, hubs included)
    stride = max(1, int(order.size // 2048))
    seeds = np.sort(order[::stride]).astype(np.uint32)
    sample_cost = float(cost[seeds.astype(np.int64)].sum())
    # level-2 rows of those seeds: probe the visit rate on a thin row sample,
    # then size the row stride so level 2 runs ~budget_s
    rs = max(1, int(sample_cost / 2e8))
    s = rg.count_sample(seeds, row_stride=rs, lookahead=2, workers=0)
    rate = s["visits"] / max(s["l2_ms"] / 1e3, 1e-3)
    rs2 = max(1, int(sample_cost / max(rate * budget_s, 1.0)))
    if rs2 < rs:
        rs = rs2
        s = rg.count_sample(seeds, row_stride=rs, lookahead=2, workers=0)
    verify_seeds_ms = s["l1_ms"] + s["l2_ms"] * rs           # all level-2 rows of the seeds
    t_est_ms = s["filter_ms"] + verify_seeds_ms * total_cost / max(sample_cost, 1.0)
    # expand_level materialises rows and zero-fills one scratch slot per visit
    # (frontier.hpp:123), which count_final_level does not: calibrate the
    # estimator once against a FULL count_triangles run on C1 (RMAT s16)
    cal = calibration() if calibrate else None
    t_full_ms = t_est_ms * (cal["factor"] if cal else 1.0)
    return {
        "value": E / (t_full_ms / 1e3) / 1e9,
        "unit": "GTEPS",
        "cores": workers,
        "kind": "reference",
        "t_full_est_ms": t_full_ms,
        "t_sample_est_ms": t_est_ms,
        "sample_wall_s": time.perf_counter() - t_wall0,
        "calibration": cal,
        "sample": (f"trimatch::count_triangles path through its public API: filter_candidates on the full "
                   f"graph ({s['filter_ms']:.0f} ms), expand_level L1 for {seeds.size} of {order.size} seeds "
                   f"(cost-stratified every {stride}th by deg(u)*|N(u)>u|, {s['l1_ms']:.0f} ms), expand_level L2 "
                   f"(final level, accept+look-ahead+has_edge) on every {rs}th of {s['l1_rows']} L1 rows "
                   f"({s['visits']} visits, {s['l2_ms']:.0f} ms); extrapolated x{rs} rows and x"
                   f"{total_cost / max(sample_cost, 1):.1f} seed cost; OpenMP workers={workers}"),
    }


def host_graph(cfg):
    """Host CSR for the CPU arms: generator + build restated in oracle/ (the
    CSR equals trimatch::build_graph's, tests/test_oracle.py)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_ctypes import Oracle
    o = Oracle()
    kind, scale, param = cfg[0], cfg[1], cfg[2]
    pairs = o.gen_er(scale, param) if kind == "er" else o.gen_rmat(scale, param, kind == "kron")
    off, nb, E, _, _ = o.build_graph(pairs, 1 << scale)
    return off, nb, E


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[a.config]
    off, nb, E = host_graph(cfg)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_ctypes import Ref
    rg = Ref().graph(off, nb)
    vals = []
    last = None
    budget = max(2.0, min(a.cpu_budget_s, 150.0 / max(1, a.steps + a.warmup)))
    for i in range(a.warmup + a.steps):
        r = reference_cpu_sample(off, nb, budget, E, rg)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtrimatch_ref.so not built"}))
            return
        if i >= a.warmup:
            vals.append(r["value"])
        last = r
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "triangle-count GTEPS (|E|/time)", "value": v, "unit": "GTEPS",
        "n_gpus": 0, "steps": a.steps, "warmup": a.warmup, "ms_per_step": E / (v * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg[4], "config": a.config, "num_edges": int(E), "num_vertices": int(off.size - 1)},
        "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": last["cores"], "kind": "reference",
                         "sample": last["sample"]},
        "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measured_reference_counts(configs=("C1", "C2")):
    """The reference's own trimatch::count_triangles (oracle/_ref, all host
    cores, lookahead=2) timed in full -- best of 3 -- on the configs where it
    finishes in seconds (matcher.cpp:301-303)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_ctypes import REF_SO, Ref
    if not os.path.exists(REF_SO):
        return None
    out = {}
    for name in configs:
        off, nb, E = host_graph(CONFIGS[name])
        rg = Ref().graph(off, nb)
        best = None
        T = 0
        for _ in range(3):
            t0 = time.perf_counter()
            T = rg.count_triangles(lookahead=2, workers=0)
            dt = (time.perf_counter() - t0) * 1e3
            best = dt if best is None else min(best, dt)
        out[name] = {"ms": best, "gteps": E / (best / 1e3) / 1e9, "triangles": int(T), "num_edges": int(E),
                     "cores": os.cpu_count(), "runs": 3, "stat": "best of 3"}
    return out


def build_inputs_sha256(root):
    """sha256 over the library's build inputs (csrc sources, headers,
    Makefile, include/): the same sources build the same kernels, while the
    .so itself is not byte-reproducible across clean builds."""
    import hashlib
    h = hashlib.sha256()
    for d in (os.path.join(root, "paper_1909_02127_b200", "csrc"), os.path.join(root, "include")):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cu", ".cuh", ".h", ".hpp", ".cpp")) or name == "Makefile":
                h.update(name.encode())
                with open(os.path.join(d, name), "rb") as f:
                    h.update(f.read())
    return h.hexdigest()


def lib_sha256():
    import hashlib
    h = hashlib.sha256()
    with open(os.path.join(ROOT, "paper_1909_02127_b200", "libtcb200.so"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def measured_traffic(config: str, kernel: str):
    """DRAM bytes per launch of the dominant kernel from the ncu capture made
    for THIS build (profiles/ncu_traffic_<config>.json, written by
    tools/ncu_traffic.py with the sha256 of the library's build inputs); None
    when stale/absent."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except Exception:
        return None, "absent"
    if d.get("src_sha256") != build_inputs_sha256(ROOT):
        return None, f"stale ({path} measured another build)"
    k = d.get("kernels", {}).get(kernel)
    if not k:
        return None, f"kernel {kernel} not in {path}"
    return k, "measured (ncu --set full, this build)"


# ---------------------------------------------------------------------------
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_1909_02127_b200 as tc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TCB_BENCH_SHARE_GPU=1 (plumbing check only): every rank on cuda:0
    share = os.environ.get("TCB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        # torch.distributed is the rendezvous only (gloo: NCCL id, barriers,
        # max over ranks); the count's allreduce is the library's own NCCL
        # communicator on the count stream (tc_count_allreduce)
        dist.init_process_group("gloo")
        from paper_1909_02127_b200 import dist as tdist
        comm = tdist.init_comm(local)
    cfg = CONFIGS[a.config]
    kind, scale, param, per_vertex, desc = cfg
    per_vertex = per_vertex and not a.no_per_vertex
    n = 1 << scale
    stream = torch.cuda.Stream(dev)  # a real stream: the handle's work and the events share it

    # ---- input: deterministic synthetic edge list generated on the device ----
    m = tc.gen_num_edges(gen_kind(tc, kind), scale, param)
    with torch.cuda.stream(stream):
        pairs = torch.empty(2 * m, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    tc.generate(gen_kind(tc, kind), scale, param, out=pairs, device=local)
    rep = tc.BuildReport()
    g = tc.build_graph_from_pairs(pairs, n, rep, device=local, m=m)
    build_ms = g.build_ms
    del pairs
    torch.cuda.empty_cache()
    E = g.num_edges()
    g.set_stream(stream.cuda_stream)

    with torch.cuda.stream(stream):
        total = torch.zeros(1, dtype=torch.int64, device=dev)
        pv = torch.zeros(n, dtype=torch.int64, device=dev) if per_vertex else None
    torch.cuda.synchronize()
    opts = tc.MatchOptions(per_vertex=per_vertex)

    def step(stats=False, work=False):
        if comm is not None:
            return comm.count_into(g, total, pv, opts, stats=stats)
        return tc.count_triangles_into(g, total, pv, opts, stats=stats, work_counters=work)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    # N=1: the whole count (plan + joins + row pass + outputs, ~15 kernels, no
    # host synchronisation, no allocation at steady state) is captured once
    # into a CUDA graph and replayed per step -- the launch overhead of the
    # small configs goes away, the work per step is unchanged
    cgraph, launch_mode = None, "direct launches"
    if world == 1 and not a.no_graph:
        try:
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=stream, capture_error_mode="relaxed"):
                step()
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for _ in range(2):
                    cg.replay()
            torch.cuda.synchronize()
            cgraph, launch_mode = cg, "CUDA graph replay of one whole count per step"
        except Exception as e:  # reported, then direct launches
            launch_mode = f"direct launches (graph capture failed: {repr(e)[:120]})"
            torch.cuda.synchronize()

    def timed_step():
        if cgraph is not None:
            cgraph.replay()
        else:
            step()

    # L2 rule: C3..C5 inputs are far larger than the 126 MB L2; for C1/C2
    # (whose oriented graph could stay L2-resident) a 512 MB buffer is written
    # between the timed steps and each step is timed on its own event pair
    flush = a.config in ("C1", "C2")
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)] \
        if flush else []
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(a.steps):
            if flush:
                scrub.fill_(i & 0xff)
                evs[i][0].record(stream)
            timed_step()
            if flush:
                evs[i][1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = (sum(x.elapsed_time(y) for x, y in evs) if flush else ev0.elapsed_time(ev1)) / a.steps
    if world > 1:
        ms = tdist.max_over_ranks(ms)
    T = int(total.item())
    # per-kernel device times: the same K steps again, CUDA events recorded by
    # the library around every join kernel on the launch stream (a stats call
    # also synchronises once at its end, so this is a second timed region,
    # not the headline one), and the work counters
    stats = [step(stats=True) for _ in range(max(3, a.steps))]
    sw = tc.count_triangles_into(g, total, pv, tc.MatchOptions(per_vertex=per_vertex, part_index=rank,
                                                               part_count=world),
                                 stats=True, work_counters=True)
    join_ms = float(np.mean([s_["join_ms"] for s_ in stats]))
    if world > 1:
        join_ms = tdist.max_over_ranks(join_ms)
    launches = int(sw["kernel_launches"]) * a.steps

    # ---- e2e: drop-in count_triangles(const Graph&) with host buffers ----
    # the host Graph = the symmetric CSR (exported once); pinned (the contract)
    # and pageable (a caller's std::vector / numpy arrays) legs
    ro_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    nb_h = torch.empty(max(2 * E, 1), dtype=torch.int32, pin_memory=True)
    g.export_csr(ro_h, nb_h)
    tot_h = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    pv_h = torch.zeros(n, dtype=torch.int64, pin_memory=True) if per_vertex else None

    link_gbps = None
    if E:
        tmp = torch.empty_like(nb_h, device=dev)
        rates = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tmp.copy_(nb_h, non_blocking=True)
            torch.cuda.synchronize()
            rates.append(nb_h.numel() * 4 / (time.perf_counter() - t0) / 1e9)
        link_gbps = max(rates)
        del tmp

    def e2e_step(ro, nb, tot_out, pv_out):
        ge = tc.graph_from_csr(ro, nb, n, E, device=local)          # H2D + orientation + in-edge index
        if comm is not None:
            comm.count_into(ge, tot_out, pv_out, opts, sync=True)  # count + allreduce + D2H
        else:
            tc.count_triangles_into(ge, tot_out, pv_out, opts, sync=True)  # count + D2H
        del ge

    def time_e2e(ro, nb, tot_out, pv_out, steps):
        e2e_step(ro, nb, tot_out, pv_out)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            e2e_step(ro, nb, tot_out, pv_out)
        torch.cuda.synchronize()
        e = (time.perf_counter() - t0) * 1e3 / steps
        return tdist.max_over_ranks(e) if world > 1 else e

    e2e_ms = time_e2e(ro_h, nb_h, tot_h, pv_h, a.e2e_steps)
    assert int(tot_h[0]) == T, (int(tot_h[0]), T)
    # pageable leg: plain numpy arrays
    ro_p = ro_h.numpy().view(np.uint64).copy()
    nb_p = nb_h.numpy().view(np.uint32).copy()
    tot_p = np.zeros(1, np.uint64)
    pv_p = np.zeros(n, np.uint64) if per_vertex else None
    e2e_pg_ms = time_e2e(ro_p, nb_p, tot_p, pv_p, max(1, a.e2e_steps - 1))
    assert int(tot_p[0]) == T
    del ro_p, nb_p

    h2d = 8 * (n + 1) + 4 * 2 * E
    d2h = 8 + (8 * n if per_vertex else 0)

    peak, peak_kind = peaks()
    alg_bytes = sw["alg_bytes"]          # this rank's share (the parts sum to the graph's B_alg)
    impl_bytes = sw["probe_bytes"]
    cta_bytes = sw["cta_bytes"]
    kms = {k: float(np.mean([s_[k + "_ms"] for s_ in stats])) for k in ("warp", "small", "cta", "dense", "rows")}
    cta_ms = kms["cta"]
    if world > 1:
        ab = torch.tensor([alg_bytes, impl_bytes, cta_bytes], dtype=torch.float64)
        dist.all_reduce(ab)
        alg_bytes, impl_bytes, cta_bytes = float(ab[0]), float(ab[1]), float(ab[2])
        cta_ms = tdist.max_over_ranks(cta_ms)
    # roofline of the dominant kernel (k_join_cta): its algorithmic bytes per
    # launch / its average launch duration (library CUDA events, above)
    achieved = cta_bytes / (cta_ms / 1e3) / 1e9 / max(1, world) if cta_ms > 0 else 0.0
    phase_achieved = impl_bytes / (join_ms / 1e3) / 1e9 / max(1, world) if join_ms > 0 else 0.0
    traffic, traffic_src = measured_traffic(a.config, "k_join_cta")
    line = {
        "metric": "triangle-count GTEPS (|E|/time)",
        "value": E / (ms / 1e3) / 1e9,
        "unit": "GTEPS",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {
            "workload": desc, "config": a.config, "generator": f"{kind} scale={scale} param={param} (SURVEY 8d splitmix)",
            "num_vertices": n, "num_edges": int(E), "raw_edges": int(m), "triangles": T,
            "per_vertex": per_vertex,
            "parallelism": (f"pivot ranges x{world} + one NCCL allreduce (tc_count_allreduce)" if world > 1
                            else "1 GPU"),
            "l2": ("L2 flushed between timed steps (512 MB written), each step timed on its own events" if flush
                   else "inputs larger than L2 (oriented CSR + in-edge index + masks >> 126 MB); no flush"),
            "launch": launch_mode,
            "build_ms": build_ms, "self_loops_removed": rep.self_loops_removed,
            "duplicate_entries_removed": rep.duplicate_entries_removed,
        },
        "e2e": {"value": E / (e2e_ms / 1e3) / 1e9, "unit": "GTEPS", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "h2d_link_gbps": link_gbps,
                "h2d_floor_ms": (h2d / link_gbps / 1e6) if link_gbps else None,
                "path": "tc_graph_from_csr(host pinned CSR) + tc_count(host outputs)",
                "pageable": {"value": E / (e2e_pg_ms / 1e3) / 1e9, "ms_per_step": e2e_pg_ms,
                             "path": "the same from pageable numpy arrays (a caller's std::vector)"}},
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic["dram_bytes"] if traffic else None, "traffic_source": traffic_src,
            "peak_kind": peak_kind,
            "kernel": "k_join_cta (sparse advance + fused SMEM join, the dominant kernel)",
            "model": "k_join_cta algorithmic bytes per launch: 2 B per sparse hot candidate + 4 B per cold "
                     "candidate + 32 B per item (its 32-byte in-edge item record) + 1 B per per-vertex "
                     "mask chunk + 4 B per pivot member and 16 B per CTA segment",
            "bytes_per_launch": cta_bytes, "kernel_ms": cta_ms,
            "kernels_ms": kms,
            "join_phase": {"achieved": phase_achieved, "frac": phase_achieved / peak, "bytes_per_step": impl_bytes,
                           "join_ms": join_ms,
                           "model": "all join kernels + row pass: 2 B per hot candidate + 4 B per cold candidate "
                                    "+ 28 B per in-edge + per-vertex masks written and read + counters"},
            "wedges_probed": sw["wedges"],
            "wedge_stream_equiv": {"B_alg": alg_bytes, "W": sw["dag_W"],
                                   "ratio": alg_bytes / (join_ms / 1e3) / 1e9 / peak / max(1, world),
                                   "note": "SURVEY 8d B_alg = 4W + 12|E+| + 8(|V|+1) + 8|V| over the join time: "
                                           "counts W wedge reads the pivot join never makes (J << W), so it "
                                           "is a model-equivalent rate, not a bandwidth"},
        },
        "phases_ms": {"frontier": float(np.mean([s_["frontier_ms"] for s_ in stats])), "join": join_ms,
                      "reduce": float(np.mean([s_["reduce_ms"] for s_ in stats]))},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if traffic:
        line["roofline"]["traffic_kernel_ms"] = traffic.get("ms")
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            ro_np = ro_h.numpy().view(np.uint64)
            nb_np = nb_h.numpy().view(np.uint32)[: 2 * E]
            cb = reference_cpu_sample(ro_np, nb_np, a.cpu_budget_s, E)
            if cb is not None:
                cb["kind"] = "reference"
                cb["value_is"] = ("extrapolated: the full reference count at this config does not finish "
                                  "(~2.6e12 visits); bounded sample + calibration, see sample")
                cb["measured"] = measured_reference_counts()
            line["cpu_baseline"] = cb
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": repr(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
