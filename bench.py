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
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--n-per-gpu", type=int, default=None, help="override the per-GPU code count (cfg4)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-s", type=float, default=20.0, help="CPU work budget of the baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", type=int, default=0, help="Quick ADC scan engine: 0 auto, 1 PRMT, 2 tcgen05")
    ap.add_argument("--sample-div", type=int, default=0, help="threshold sample = 1/N of the tiles (0: library default)")
    return ap.parse_args()


# --------------------------------------------------------------------- data
CFG4_PER_GPU = 125_000_000   # BASELINE cfg4: 1e9 codes sharded over 8 GPUs


def make_data_device(cfg_name: str, rank: int, world: int, ctx, n_per_gpu=None):
    """cfg4: each rank generates and encodes its own 125M-code shard on the GPU
    (Philox rows -> exact encode kernel); prefix = global rows [0, init_count)."""
    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS[cfg_name]
    n = n_per_gpu or CFG4_PER_GPU
    books, codes, prefix, queries = G.make_quick_adc_shard(
        cfg_name, rank, world, lambda b: P.DeviceQuantizer(P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], b), ctx),
        n=n, device=f"cuda:{ctx.device}")
    return cfg, books, codes, queries, prefix


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


CPU_CODE_SAMPLE = 4_000_000


def cpu_baseline(cfg, books, codes, queries, budget_s: float, n_full: int | None = None):
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
            "sample": f"{nq} of {queries.shape[0]} queries over "
                      + (f"all {codes.shape[0]} codes" if n_full is None else
                         f"the first {codes.shape[0]} of {n_full} codes (evals/s is per (query, code))")
                      + f" (oracle/pqscan_oracle.py, fork pool x{cores}); single-core {per_q * 1e3:.1f} ms/query"}


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
    n_full = None
    if args.config == "cfg3":
        # the index is built on the GPU (data preparation, untimed); the timed
        # path is the oracle's query_ivf on the host cores
        import torch

        import paper_1712_02912_b200 as P

        ctx = P.Context(0)
        cfg, books, coarse, sizes, codes, ids, queries = make_ivf(args, ctx, torch.device("cuda", 0))
        vals = []
        for s in range(args.warmup + args.steps):
            base = cpu_baseline_ivf(books, coarse.cpu().numpy(), sizes, codes.cpu().numpy(), ids.cpu().numpy(),
                                    queries, cfg["nprobe"], cfg["r"],
                                    max(2.0, args.cpu_sample_s / max(args.steps, 1)))
            if s >= args.warmup:
                vals.append(base["value"])
        value = statistics.median(vals)
        print(json.dumps({
            "impl": "reference", "metric": metric_name("cfg3"), "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded stand-in; index built on the GPU, untimed)",
            "config": {"workload": "IVFADC K=65536, residual PQ 8x8, nprobe 64", "baseline_config_index": 3},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": base["cores"], "kind": "port",
                             "sample": base["sample"]},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
            flush=True)
        return
    if args.config == "cfg4":
        # host-generated sample of a shard (same distribution; the full shard
        # is GPU-generated in the "ours" arm); evals/s is per (query, code)
        from paper_1712_02912_b200 import datagen as G

        n_full = args.n_per_gpu or CFG4_PER_GPU
        cfg = G.CONFIGS["cfg4"]
        books, codes, queries = G.make_exhaustive("cfg4", n=CPU_CODE_SAMPLE)
    else:
        cfg, books, codes, queries, _ = make_data(args.config, 0)
    base = None
    vals = []
    for s in range(args.warmup + args.steps):
        base = cpu_baseline(cfg, books, codes, queries, budget_s=max(2.0, args.cpu_sample_s / max(args.steps, 1)),
                            n_full=n_full)
        if s >= args.warmup:
            vals.append(base["value"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (n_full or codes.shape[0]) * queries.shape[0] / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if cfg["b"] == 4 else "f64",
        "data": "synthetic (seeded stand-in for the BASELINE config; see DESIGN.md)",
        "config": config_dict(args.config, cfg, world, args.n_per_gpu),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": base["cores"], "kind": "port",
                         "sample": base["sample"]},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(name, cfg, world, n_per_gpu=None):
    n_per = cfg["N"] if name != "cfg4" else (n_per_gpu or CFG4_PER_GPU)
    d = {"workload": {"cfg0": "exhaustive PQ 8x8 float ADC", "cfg1": "Quick ADC PQ 16x4 exhaustive",
                      "cfg2": "high-dim PQ 64x8 float ADC",
                      "cfg4": "billion-scale sharded Quick ADC PQ 16x4 (d=96), one 125M-code shard per GPU"}[name],
         "baseline_config_index": int(name[-1]), "N_per_gpu": n_per, "N_total": n_per * world,
         "queries": cfg["Q"], "d": cfg["d"], "m": cfg["m"], "b": cfg["b"], "r": cfg["r"],
         "parallelism": f"shard{world}" if world > 1 else "single", "l2": "flushed between timed steps (256 MB write)"}
    if cfg["b"] == 4:
        d["init_count"] = cfg["init_count"]
    return d


# --------------------------------------------------------------- IVF (cfg3)
_IVF = {}


def _cpu_ivf_query(qi):
    from oracle import pqscan_oracle as O

    d = _IVF
    O.query_ivf(d["coarse"], d["books"], d["lists_codes"], d["lists_ids"], d["queries"][qi], d["ma"], d["r"])
    return qi


def cpu_baseline_ivf(books, coarse, sizes, codes, ids, queries, ma, r, budget_s):
    """Oracle query_ivf (ivf.py:148-196) in a fork pool over all host cores."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    offs = np.concatenate([[0], np.cumsum(sizes)])
    _IVF.update(books=books, coarse=coarse, queries=queries, ma=ma, r=r,
                lists_codes=[codes[offs[c]:offs[c + 1]] for c in range(len(sizes))],
                lists_ids=[ids[offs[c]:offs[c + 1]] for c in range(len(sizes))])
    t0 = time.perf_counter()
    _cpu_ivf_query(0)
    per_q = time.perf_counter() - t0
    nq = min(queries.shape[0], max(cores, (int(budget_s / max(per_q, 1e-3)) // cores) * cores))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        pool.map(_cpu_ivf_query, range(nq), chunksize=1)
        wall = time.perf_counter() - t0
    # exact evaluation count of the sampled queries (untimed): sizes of their probed lists
    from oracle import pqscan_oracle as O

    cells, _ = O.nearest_k(queries[:nq].astype(np.float64), np.asarray(coarse, np.float32).astype(np.float64), ma)
    evals = float(np.asarray(sizes)[cells].sum())
    return {"value": evals / wall, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"{nq} of {queries.shape[0]} queries, nprobe {ma}, full index (oracle query_ivf, fork pool "
                      f"x{cores}); {evals:.3e} probed codes; single-core {per_q * 1e3:.1f} ms/query"}


def make_ivf(args, ctx, dev):
    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS["cfg3"]
    books, coarse, sizes, codes, ids, queries = G.make_ivf_device(
        "cfg3", lambda b: P.DeviceQuantizer(P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], b), ctx),
        n=args.n_per_gpu, device=dev)
    return cfg, books, coarse, sizes, codes, ids, queries


def run_ivf(args):
    """cfg3 (IVFADC): one index per GPU, queries sharded across ranks (each
    rank searches its own 10k-query batch against a replica of the index:
    weak scaling, no exchange -- "replicas")."""
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

    ctx = P.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    t_build = time.perf_counter()
    cfg, books, coarse, sizes, codes, ids, queries = make_ivf(args, ctx, dev)
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    ivf = P.DeviceIvf.from_arrays(pq, coarse, sizes, codes, ids, ctx=ctx)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    ma, r = cfg["nprobe"], cfg["r"]
    q_dev = torch.from_numpy(queries).to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for _ in range(args.warmup):
        ivf.search(q_dev, ma, r)
    torch.cuda.synchronize()
    launches0 = ctx.stat(_lib.STAT_LAUNCHES)
    clocks = ClockSampler(local)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    scan_ns, evals = [], []
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for s in range(args.steps):
        flush.zero_()
        starts[s].record(stream)
        ivf.search(q_dev, ma, r)
        ends[s].record(stream)
        scan_ns.append(ctx.stat(_lib.STAT_LAST_SCAN_NS))
        evals.append(ctx.stat(_lib.STAT_LAST_EVALS))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.stat(_lib.STAT_LAUNCHES) - launches0
    cand_max, cand_tot = ctx.stat(_lib.STAT_LAST_MAX_CAND), ctx.stat(_lib.STAT_LAST_CAND_TOTAL)
    total_ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    evals_step = float(evals[-1])
    t = torch.tensor([total_ms, evals_step], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist

        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ev = t[1:].clone()
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
        total_ms, evals_all = float(tm.item()), float(ev.item())
    else:
        evals_all = evals_step
    ms_per_step = total_ms / args.steps
    value = evals_all / (ms_per_step / 1e3)
    # e2e: host queries in, host results out, through the drop-in API call
    # (pinned caller-owned buffers, reused across calls)
    q_pin = torch.from_numpy(np.ascontiguousarray(queries)).pin_memory().numpy()
    nq_h = queries.shape[0]
    o_pin = (torch.empty((nq_h, r), dtype=torch.float64).pin_memory().numpy(),
             torch.empty((nq_h, r), dtype=torch.int64).pin_memory().numpy(),
             torch.empty((nq_h,), dtype=torch.int32).pin_memory().numpy())
    e2e = []
    for s in range(max(args.warmup, 1) + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        ivf.search(q_pin, ma, r, out=o_pin)
        dt = (time.perf_counter() - t0) * 1e3
        if s >= max(args.warmup, 1):
            e2e.append(dt)
    e2e_total = sum(e2e)
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_total = float(tt.item())
    e2e_value = evals_all / (e2e_total / len(e2e) / 1e3)
    nq = queries.shape[0]
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    scan_ms = statistics.mean(scan_ns) / 1e6
    m = cfg["m"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = clk.get("sm_mhz") or 1965.0
    lut_peak = sm_count * 32 * f_mhz * 1e6 / 1e9
    lut_rate = evals_step * m / (scan_ms / 1e3) / 1e9
    hbm_alg = int(codes.shape[0]) * (m + 4)  # list-major: every list's codes + V once per launch
    hbm_peak = peaks.get("hbm_gbs", 6553.6)
    line = {
        "metric": metric_name("cfg3"), "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded stand-in for the BASELINE config, index built on the GPU; see DESIGN.md)",
        "config": {"workload": "IVFADC K=65536, residual PQ 8x8, nprobe 64", "baseline_config_index": 3,
                   "N_per_gpu": int(codes.shape[0]), "queries_per_gpu": nq, "K": int(coarse.shape[0]),
                   "nprobe": ma, "m": m, "b": cfg["b"], "r": r, "d": cfg["d"],
                   "evals_per_step_per_gpu": evals_step,
                   "parallelism": f"query-shard replicas x{world}" if world > 1 else "single",
                   "l2": "flushed between timed steps (256 MB write); index 1.6 GB > L2",
                   "index_build_s": t_build},
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": queries.nbytes,
                "d2h_bytes_per_step": nq * r * 16 + nq * 4},
        "gpu_launches": launches,
        "candidates": {"max_per_query": cand_max, "mean_per_query": cand_tot / nq,
                       "reranked_per_query": ctx.stat(_lib.STAT_LAST_RERANK_TOTAL) / nq,
                       "list_scan_slot_utilization": (ctx.stat(_lib.STAT_LAST_EVALS) /
                                                      max(1, ctx.stat(_lib.STAT_LAST_SLOT_EVALS)))},
        "clocks": clk,
        "roofline": {"bound": "lut", "achieved": lut_rate, "peak": lut_peak, "unit": "Glookup/s",
                     "frac": lut_rate / lut_peak, "traffic": _ncu_traffic("ivf_list_kernel"),
                     "traffic_note": "DRAM bytes of one list-scan launch from the committed ncu capture (profiles/r01_ivf_cfg3.md); the excess over the algorithmic bytes is the per-(list, query) staging of the 8 KB query tables",
                     "kernel": "ivf_list_kernel (list-major, smem LUT)",
                     "per_unit": f"{m} table lookups per probed (query, code); {evals_step:.3e} per launch",
                     "peak_source": f"shared-memory LUT rate {sm_count} SM x 32 lookups/clk x {f_mhz:.0f} MHz",
                     "hbm": {"algorithmic_bytes": hbm_alg, "achieved_GBs": hbm_alg / (scan_ms / 1e3) / 1e9,
                             "peak_GBs": hbm_peak, "frac": hbm_alg / (scan_ms / 1e3) / 1e9 / hbm_peak},
                     "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step},
        "impl": "ours",
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_ivf(books, coarse.cpu().numpy(), sizes, codes.cpu().numpy(),
                                                ids.cpu().numpy(), queries, ma, r, args.cpu_sample_s)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _ncu_traffic(kernel: str):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(kernel, {}).get("bytes")
    except (OSError, ValueError):
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "cfg3":
        run_ivf(args)
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

    ctx = P.Context(local)
    if args.config == "cfg4":
        cfg, books, codes, queries, prefix = make_data_device(args.config, rank, world, ctx, args.n_per_gpu)
    else:
        cfg, books, codes, queries, prefix = make_data(args.config, rank)
    nq, n, r = queries.shape[0], codes.shape[0], cfg["r"]
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_option(_lib.OPT_SCAN4_ENGINE, args.engine)
    if args.sample_div:
        ctx.set_option(_lib.OPT_SAMPLE_DIV, args.sample_div)
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
    # caller-owned pinned result buffers, reused across calls (the D2H lands in them directly)
    o_pin = (torch.empty((nq, r), dtype=torch.uint8 if cfg["b"] == 4 else torch.float64).pin_memory().numpy(),
             torch.empty((nq, r), dtype=torch.int64).pin_memory().numpy(),
             torch.empty((nq,), dtype=torch.int32).pin_memory().numpy())
    e2e_ms = []
    for s in range(max(args.warmup, 1) + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            # the drop-in batched API on host arrays: H2D/D2H inside the C ABI call
            if cfg["b"] == 4:
                out = searcher.db.qadc_search(searcher.dq, q_pin.numpy(), cfg["init_count"], r, out=o_pin)
            else:
                out = searcher.db.adc_search(searcher.dq, q_pin.numpy(), r, out=o_pin)
        else:
            d_, i_, c_ = searcher.search(q_pin.to(dev, non_blocking=True), r)
            if s == 0:
                o_sh = tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in (d_, i_, c_))
            for dst, src in zip(o_sh, (d_, i_, c_)):
                dst.copy_(src, non_blocking=True)
            out = o_sh
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
                    "traffic_note": "DRAM bytes of the filter launches of one search from the committed ncu capture (profiles/r01_final_cfg1.md)",
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
        "config": config_dict(args.config, cfg, world, args.n_per_gpu),
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "candidates": {"max_per_query": cand_max, "mean_per_query": cand_tot / nq,
                       "reranked_per_query": (ctx.stat(_lib.STAT_LAST_RERANK_TOTAL) / nq) if cfg["b"] == 8 else None,
                       "note": "codes surviving the certified threshold filter (float: the exact re-score sees "
                               "only those within the tightened bound)"},
        "clocks": clk,
        "roofline": roofline,
        "impl": "ours",
    }
    if not args.no_cpu_baseline and world == 1:
        if isinstance(codes, np.ndarray):
            line["cpu_baseline"] = cpu_baseline(cfg, books, codes, queries, args.cpu_sample_s)
        else:  # device-generated shard: the oracle runs on a host copy of its first codes
            sample = codes[:CPU_CODE_SAMPLE].cpu().numpy()
            line["cpu_baseline"] = cpu_baseline(cfg, books, sample, queries, args.cpu_sample_s, n_full=n)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
