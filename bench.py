#!/usr/bin/env python3
"""Benchmark: ADC distance evals/s (codes x queries) on B200.

Default workload (N=1): BASELINE.json configs[1] -- Quick ADC, PQ 16x4 over a
seeded d=128 Gaussian-mixture stand-in, N=1,000,000 codes, 1,000 queries,
top-100, init_count 200.  A "step" is one pass of the hot path over the
whole query batch: tables -> Quick ADC params -> threshold sample -> PRMT
scan -> (bin, id) top-100 for all 1,000 queries.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1]
                  [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling -- every rank owns its own
1M-code shard of one global list (ids offset by rank), all ranks scan the
same queries with the GLOBAL Quick ADC prefix, the per-rank top-100 lists are
all-gathered over NCCL and merged on the device (pqs_merge_topr).

--impl reference: the reference's CPU path of the same workload on the
host's cores (the oracle port of pqscan, oracle/pqscan_oracle.py, in a fork
process pool), rank 0 only.
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

L2_FLUSH_BYTES = 256 << 20   # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-s", type=float, default=20.0, help="CPU work budget of the baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", type=int, default=0, help="Quick ADC scan engine: 0 auto, 1 PRMT, 2 tcgen05")
    return ap.parse_args()


# --------------------------------------------------------------------- data
def make_data(cfg_name: str, rank: int):
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS[cfg_name]
    books, codes, queries = G.make_exhaustive(cfg_name, shard=rank)
    prefix = None
    if cfg["b"] == 4:
        prefix = codes[:cfg["init_count"]] if rank == 0 else \
            G.encode(books, G.rows(cfg, 1712, 0, cfg["init_count"], stream=1))
    return cfg, books, codes, queries, prefix


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
_CPU = {}


def _cpu_query(qi):
    from oracle import pqscan_oracle as O

    d = _CPU
    t = O.compute_tables(d["books"], d["queries"][qi])
    if d["b"] == 4:
        O.qadc_scan(d["codes"], d["ids"], t, d["init"], d["r"])
    else:
        O.scan(d["codes"], d["ids"], t, d["r"])
    return qi


def cpu_baseline(cfg, books, codes, queries, budget_s: float):
    """Oracle port of the reference CPU path, fork process pool over all host
    cores (threads do not scale: GIL, SURVEY finding 8)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _CPU.update(books=books, codes=codes, queries=queries, ids=np.arange(codes.shape[0], dtype=np.int64),
                b=cfg["b"], init=cfg.get("init_count", 200), r=cfg["r"])
    t0 = time.perf_counter()
    _cpu_query(0)  # warm-up (cli._run_timed, cli.py:266-276)
    per_q = time.perf_counter() - t0
    nq = int(max(cores, min(queries.shape[0], round(budget_s / max(per_q, 1e-3)))))
    nq = min(queries.shape[0], max(cores, (nq // cores) * cores))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        pool.map(_cpu_query, range(nq), chunksize=1)
        wall = time.perf_counter() - t0
    evals = nq * codes.shape[0]
    return {"value": evals / wall, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"{nq} of {queries.shape[0]} queries over all {codes.shape[0]} codes "
                      f"(oracle/pqscan_oracle.py, fork pool x{cores}); single-core {per_q * 1e3:.1f} ms/query"}


# ------------------------------------------------------------------ driver
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def metric_name(cfg_name):
    return "ADC distance evals/sec (codes x queries)"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, books, codes, queries, _ = make_data(args.config, 0)
    base = None
    vals = []
    for s in range(args.warmup + args.steps):
        base = cpu_baseline(cfg, books, codes, queries, budget_s=max(2.0, args.cpu_sample_s / max(args.steps, 1)))
        if s >= args.warmup:
            vals.append(base["value"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": codes.shape[0] * queries.shape[0] / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if cfg["b"] == 4 else "f64",
        "data": "synthetic (seeded stand-in for the BASELINE config; see DESIGN.md)",
        "config": config_dict(args.config, cfg, world),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": base["cores"], "kind": "port",
                         "sample": base["sample"]},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(name, cfg, world):
    d = {"workload": {"cfg0": "exhaustive PQ 8x8 float ADC", "cfg1": "Quick ADC PQ 16x4 exhaustive",
                      "cfg2": "high-dim PQ 64x8 float ADC"}[name],
         "baseline_config_index": int(name[-1]), "N_per_gpu": cfg["N"], "N_total": cfg["N"] * world,
         "queries": cfg["Q"], "d": cfg["d"], "m": cfg["m"], "b": cfg["b"], "r": cfg["r"],
         "parallelism": f"shard{world}" if world > 1 else "single", "l2": "flushed between timed steps (256 MB write)"}
    if cfg["b"] == 4:
        d["init_count"] = cfg["init_count"]
    return d


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import _lib

    cfg, books, codes, queries, prefix = make_data(args.config, rank)
    nq, n, r = queries.shape[0], codes.shape[0], cfg["r"]
    ctx = P.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_option(_lib.OPT_SCAN4_ENGINE, args.engine)
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    from paper_1712_02912_b200.sharded import ShardedSearch

    n_total = n * world
    if cfg["b"] == 4:
        if prefix is None:
            prefix = codes[:cfg["init_count"]]
        searcher = ShardedSearch.quick_adc(codes, rank, world, n_total, prefix, pq, cfg["init_count"], ctx=ctx)
    else:
        searcher = ShardedSearch.float_adc(codes, rank, world, n_total, pq, ctx=ctx)
    q_dev = torch.from_numpy(queries).to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step_device():
        return searcher.search(q_dev, r)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    launches0 = ctx.stat(_lib.STAT_LAUNCHES)
    clocks = ClockSampler(local)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    scan_ns = []
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for s in range(args.steps):
        flush.zero_()
        starts[s].record(stream)
        step_device()
        ends[s].record(stream)
        scan_ns.append(ctx.stat(_lib.STAT_LAST_SCAN_NS))
    cand_max, cand_tot = ctx.stat(_lib.STAT_LAST_MAX_CAND), ctx.stat(_lib.STAT_LAST_CAND_TOTAL)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.stat(_lib.STAT_LAUNCHES) - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    evals_per_step = nq * n * world
    value = evals_per_step / (ms_per_step / 1e3)

    # ---- e2e through the public API with host buffers (pinned), H2D + D2H inside
    q_pin = torch.from_numpy(queries).pin_memory()
    e2e_ms = []
    for s in range(max(args.warmup, 1) + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            # the drop-in batched API on host arrays: H2D/D2H inside the C ABI call
            if cfg["b"] == 4:
                out = searcher.db.qadc_search(searcher.dq, q_pin.numpy(), cfg["init_count"], r)
            else:
                out = searcher.db.adc_search(searcher.dq, q_pin.numpy(), r)
        else:
            d_, i_, c_ = searcher.search(q_pin.to(dev, non_blocking=True), r)
            out = (d_.cpu(), i_.cpu(), c_.cpu())
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if s >= max(args.warmup, 1):
            e2e_ms.append(dt)
    e2e_total = sum(e2e_ms)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = evals_per_step / (e2e_total / len(e2e_ms) / 1e3)
    h2d = queries.nbytes
    d2h = nq * r * (1 if (cfg["b"] == 4 and world == 1) else 8) + nq * r * 8 + nq * 4

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the filtered scan), live CUDA events
    scan_ms = statistics.mean(scan_ns) / 1e6
    m = cfg["m"]
    engine = ctx.stat(_lib.STAT_LAST_SCAN_ENGINE)
    work = ctx.stat(_lib.STAT_LAST_SCAN_WORK)
    lookups = float(nq) * n * m
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    lut_peak = sm_count * 32 * f_mhz * 1e6 / 1e9       # Glookup/s, shared-memory LUT rate (north star)
    lut_rate = lookups / (scan_ms / 1e3) / 1e9
    code_bytes = n * (m // 2 if cfg["b"] == 4 else m)
    hbm_alg = code_bytes + nq * m * (16 if cfg["b"] == 4 else (1 << cfg["b"]) * 4)
    hbm_peak = peaks.get("hbm_gbs", 6553.6)
    hbm = {"algorithmic_bytes": hbm_alg, "achieved_GBs": hbm_alg / (scan_ms / 1e3) / 1e9, "peak_GBs": hbm_peak,
           "frac": hbm_alg / (scan_ms / 1e3) / 1e9 / hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    lut = {"achieved": lut_rate, "peak": lut_peak, "unit": "Glookup/s", "frac": lut_rate / lut_peak,
           "per_unit": f"{m} table lookups per (query, code) evaluation; {nq} x {n} evaluations per launch",
           "peak_source": f"shared-memory LUT rate {sm_count} SM x 32 lookups/clk x median SM clock under load "
                          f"({f_mhz:.0f} MHz, nvidia-smi during the timed region)"}
    traffic_db = {}
    try:
        traffic_db = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        pass
    if engine == 2:
        # tcgen05 kind::i8 one-hot GEMM: int8 MMA ops actually issued per launch
        i8_peak = 2.0 * peaks.get("bf16_tflops", 1682.0)  # dense int8 = 2x dense bf16 (nominal 4.5 vs 2.25 P)
        achieved = work / (scan_ms / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved, "peak": i8_peak, "unit": "TOP/s (int8)",
                    "frac": achieved / i8_peak,
                    "traffic": traffic_db.get("scan4tc_kernel", {}).get("bytes"),
                    "traffic_note": "DRAM bytes per launch from the committed ncu capture (profiles/)",
                    "kernel": "scan4tc_kernel (tcgen05.mma kind::i8, M=128 N=256 K=256 per tile)",
                    "per_unit": "2 x 256 int8 MACs per (query, code) over 256-query groups and 128-code tiles "
                                f"({work:.3e} ops per launch)",
                    "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (measured cuBLAS bf16; int8 dense "
                                   "rate is 2x bf16 on B200) -- derived, not separately measured",
                    "lut_equivalent": lut, "hbm": hbm, "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step}
    else:
        roofline = {"bound": "lut", **lut, "traffic": None,
                    "kernel": {1: "scan4_kernel<16,FILTER> (PRMT register LUT)", 3: "scan8_kernel (smem LUT)"}.get(
                        engine, str(engine)),
                    "hbm": hbm, "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step}
    line = {
        "metric": metric_name(args.config), "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if cfg["b"] == 4 else "f32+f64",
        "data": "synthetic (seeded stand-in for the BASELINE config; see DESIGN.md)",
        "config": config_dict(args.config, cfg, world),
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "candidates": {"max_per_query": cand_max, "mean_per_query": cand_tot / nq,
                       "note": "codes surviving the certified threshold filter, re-scored exactly"},
        "clocks": clk,
        "roofline": roofline,
        "impl": "ours",
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, books, codes, queries, args.cpu_sample_s)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
