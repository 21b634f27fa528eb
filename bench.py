#!/usr/bin/env python3
"""Benchmark: ADC distance evals/s (codes x queries) on B200.

Default workload: BASELINE.json configs[4] -- billion-scale sharded Quick
ADC (PQ 16x4, d=96 decaying-variance Gaussian, L2-normalised), one 125M-code
shard per GPU (1e9 codes at N=8), 10,000 queries, top-100, init_count 1000
with the GLOBAL prefix.  N=1 is the largest single-GPU configuration and the
unit of the north-star scaling target; N=8 is exactly BASELINE cfg4.  A
"step" is one pass of the hot path over the whole query batch: tables ->
Quick ADC params -> threshold sample -> tcgen05 filtered scan -> (bin, id)
top-100 for all 10,000 queries (-> all-gather + merge at N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg0..cfg4]
                  [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling -- every rank owns its own
shard of one global list (ids offset by rank), all ranks scan the same
queries with the GLOBAL Quick ADC prefix, the per-rank top-100 lists are
all-gathered over NCCL and merged on the device (pqs_merge_topr).

--impl reference: the reference's own CPU implementation of the path --
`pqscan` installed unmodified from /root/reference into baseline/_ref (pip
--target; the oracle port oracle/pqscan_oracle.py only if that install is
absent) -- in a fork process pool over the host's cores, rank 0 only; every
step times all queries of a fixed-size sample of the same workload.
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
    ap.add_argument("--config", default="cfg4", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--n-per-gpu", type=int, default=None, help="override the per-GPU code count (cfg4)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-s", type=float, default=20.0, help="CPU work budget of the baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", type=int, default=0, help="Quick ADC scan engine: 0 auto, 1 PRMT, 2 tcgen05")
    ap.add_argument("--tc-chunk-tiles", type=int, default=0, help="tcgen05 Quick ADC scan: 128-code tiles per launch (0: library default)")
    ap.add_argument("--scan8-engine", type=int, default=0, help="float ADC filter: 0 auto (packed), 1 u16 lane=query, 2 packed")
    ap.add_argument("--ivf-engine", type=int, default=0, help="IVF list scan: 0 auto (packed), 1 float, 2 packed")
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
# The reference CPU path: pqscan itself when baseline/_ref holds the pip
# --target install of /root/reference (kind "reference"), else the oracle
# port (kind "port").  Fork process pool over all host cores (threads do not
# scale: GIL, SURVEY finding 8), the data inherited copy-on-write; per-query
# timing as cli._run_timed (cli.py:266-276).
_REF = {}
CPU_CODE_SAMPLE = 4_000_000


def _ref_module():
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "pqscan")):
        if p not in sys.path:
            sys.path.insert(0, p)
        import pqscan

        return pqscan, "reference"
    from oracle import pqscan_oracle as O

    return O, "port"


def _ref_setup(cfg, books, codes=None, queries=None, ivf=None):
    """Build the reference's own containers once (parent process, untimed)."""
    mod, kind = _ref_module()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _REF.clear()
    _REF.update(mod=mod, kind=kind, b=cfg["b"], r=cfg["r"], init=cfg.get("init_count", 200), queries=queries,
                books=books)
    if kind == "reference":
        pq = mod.ProductQuantizer(m=cfg["m"], b=cfg["b"], d=cfg["d"], codebooks=books)
        _REF["pq"] = pq
        if ivf is not None:
            coarse, sizes, lcodes, lids = ivf
            offs = np.concatenate([[0], np.cumsum(sizes)])
            lists = [mod.CodeList(lcodes[offs[c]:offs[c + 1]], lids[offs[c]:offs[c + 1]]) for c in range(len(sizes))]
            _REF["index"] = mod.IvfIndex(coarse=coarse, pq=pq, lists=lists)
        elif cfg["b"] == 4:
            _REF["tlist"] = mod.transpose_blocks(mod.CodeList(codes), 4)
        else:
            _REF["codelist"] = mod.CodeList(codes)
    else:
        if ivf is not None:
            coarse, sizes, lcodes, lids = ivf
            offs = np.concatenate([[0], np.cumsum(sizes)])
            _REF.update(coarse=coarse, lists_codes=[lcodes[offs[c]:offs[c + 1]] for c in range(len(sizes))],
                        lists_ids=[lids[offs[c]:offs[c + 1]] for c in range(len(sizes))])
        else:
            _REF.update(codes=codes, ids=np.arange(codes.shape[0], dtype=np.int64))
    if ivf is not None:
        _REF.update(ivf=True, ma=cfg["nprobe"])
    return kind


def _ref_probes(queries, coarse, ma):
    """The probed cells of a query sample (evaluation accounting, outside the
    timed window): the reference's own nearest_k (_dist.py:42-67) when it is
    installed, else the oracle's."""
    q64 = np.asarray(queries, np.float64)
    c64 = np.asarray(coarse, np.float32).astype(np.float64)
    if _REF.get("kind") == "reference":
        from pqscan._dist import nearest_k
    else:
        from oracle.pqscan_oracle import nearest_k
    return nearest_k(q64, c64, ma)[0]


def _ref_query(qi):
    """One reference query (forked worker); returns its wall time."""
    d = _REF
    q = d["queries"][qi % d["queries"].shape[0]]
    mod = d["mod"]
    t0 = time.perf_counter()
    if d["kind"] == "reference":
        if d.get("ivf"):
            mod.query_ivf(d["index"], q, d["ma"], d["r"])
        elif d["b"] == 4:
            mod.qadc_scan(d["tlist"], mod.compute_tables(d["pq"], q), d["init"], d["r"])
        else:
            mod.scan(d["codelist"], mod.compute_tables(d["pq"], q), d["r"])
    else:
        if d.get("ivf"):
            mod.query_ivf(d["coarse"], d["books"], d["lists_codes"], d["lists_ids"], q, d["ma"], d["r"])
        elif d["b"] == 4:
            mod.qadc_scan(d["codes"], d["ids"], mod.compute_tables(d["books"], q), d["init"], d["r"])
        else:
            mod.scan(d["codes"], d["ids"], mod.compute_tables(d["books"], q), d["r"])
    return time.perf_counter() - t0


def ref_run(evals_of, steps: int, warmup: int, step_budget_s: float):
    """Time the reference path: `warmup` + `steps` steps, each a fixed sample
    of queries (cores x per-core, sized from one warm-up query so a step takes
    ~step_budget_s) run in the fork pool; every query of a step is inside its
    wall-clock window.  evals_of(list of query indices) -> evaluations."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    single = _ref_query(0)                       # warm-up query (cli._run_timed)
    per_core = max(1, int(step_budget_s / max(single, 1e-3)))
    qps = cores * per_core
    nq = _REF["queries"].shape[0]
    vals, walls, per_q = [], [], []
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for s in range(warmup + steps):
            idx = [(1 + s * qps + i) % nq for i in range(qps)]
            t0 = time.perf_counter()
            times = pool.map(_ref_query, idx, chunksize=1)
            wall = time.perf_counter() - t0
            if s >= warmup:
                vals.append(evals_of(idx) / wall)
                walls.append(wall)
                per_q.extend(times)
    return {"value": statistics.median(vals), "cores": cores, "queries_per_step": qps,
            "ms_per_step": statistics.median(walls) * 1e3, "single_core_ms_per_query": statistics.median(per_q) * 1e3}


def cpu_baseline(cfg, books, codes, queries, budget_s: float, n_full: int | None = None, steps: int = 1):
    """The reference CPU path on a bounded sample (see ref_run)."""
    kind = _ref_setup(cfg, books, codes, queries)
    n = codes.shape[0]
    res = ref_run(lambda idx: len(idx) * n, steps, 0, budget_s / max(steps, 1))
    what = "pqscan (the reference, baseline/_ref)" if kind == "reference" else "oracle/pqscan_oracle.py (port)"
    return {"value": res["value"], "unit": "evals/s", "cores": res["cores"], "kind": kind,
            "sample": f"{res['queries_per_step']} queries per step over "
                      + (f"all {n} codes" if n_full is None else
                         f"the first {n} of the shard's {n_full} codes (evals/s is per (query, code))")
                      + f"; {what}, fork pool x{res['cores']}; single-core median "
                        f"{res['single_core_ms_per_query']:.1f} ms/query",
            "ms_per_step": res["ms_per_step"]}


# ------------------------------------------------------------------ driver
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def metric_name(cfg_name):
    return "ADC distance evals/sec (codes x queries)"


def _ref_line(args, world, cfg_name, cfg, res, kind, sample, dtype, config):
    return {
        "impl": "reference", "metric": metric_name(cfg_name), "value": res["value"], "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded stand-in for the BASELINE config; see DESIGN.md)",
        "config": config,
        "cpu_baseline": {"value": res["value"], "unit": "evals/s", "cores": res["cores"], "kind": kind,
                         "sample": sample},
        "e2e": {"value": res["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    step_s = max(0.5, args.cpu_sample_s / max(args.steps + args.warmup, 1))
    if args.config == "cfg3":
        # the index is built on the GPU (data preparation, untimed); the timed
        # path is the reference's query_ivf on the host cores
        import torch

        import paper_1712_02912_b200 as P

        ctx = P.Context(0)
        cfg, books, coarse, sizes, codes, ids, queries = make_ivf(args, ctx, torch.device("cuda", 0))
        coarse_h, codes_h, ids_h = coarse.cpu().numpy(), codes.cpu().numpy(), ids.cpu().numpy()
        del ctx
        kind = _ref_setup(cfg, books, queries=queries, ivf=(coarse_h, sizes, codes_h, ids_h))

        def evals_of(idx):  # exact evaluation count: sizes of the probed lists (untimed, after the step)
            cells = _ref_probes(queries[idx], coarse_h, cfg["nprobe"])
            return float(np.asarray(sizes)[cells].sum())

        res = ref_run(evals_of, args.steps, args.warmup, step_s)
        sample = (f"{res['queries_per_step']} of {queries.shape[0]} queries per step, nprobe {cfg['nprobe']}, full "
                  f"index; single-core median {res['single_core_ms_per_query']:.1f} ms/query")
        line = _ref_line(args, world, "cfg3", cfg, res, kind, sample, "f64",
                         {"workload": "IVFADC K=65536, residual PQ 8x8, nprobe 64", "baseline_config_index": 3})
        print(json.dumps(line), flush=True)
        return
    n_full = None
    if args.config == "cfg4":
        # host-generated sample of a shard (same distribution; the full shard
        # is GPU-generated in the "ours" arm); evals/s is per (query, code)
        from paper_1712_02912_b200 import datagen as G

        n_full = args.n_per_gpu or CFG4_PER_GPU
        cfg = G.CONFIGS["cfg4"]
        books, codes, queries = G.make_exhaustive("cfg4", n=CPU_CODE_SAMPLE)
    else:
        cfg, books, codes, queries, _ = make_data(args.config, 0)
    kind = _ref_setup(cfg, books, codes, queries)
    n = codes.shape[0]
    res = ref_run(lambda idx: len(idx) * n, args.steps, args.warmup, step_s)
    sample = (f"{res['queries_per_step']} queries per step over "
              + (f"all {n} codes" if n_full is None else f"the first {n} codes of a {n_full}-code shard "
                                                         "(evals/s per (query, code))")
              + f"; single-core median {res['single_core_ms_per_query']:.1f} ms/query")
    line = _ref_line(args, world, args.config, cfg, res, kind, sample, "u8" if cfg["b"] == 4 else "f64",
                     config_dict(args.config, cfg, world, args.n_per_gpu))
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
def cpu_baseline_ivf(cfg, books, coarse, sizes, codes, ids, queries, budget_s):
    """The reference query_ivf (ivf.py:148-196) on a bounded query sample."""
    kind = _ref_setup(cfg, books, queries=queries, ivf=(coarse, sizes, codes, ids))

    def evals_of(idx):  # exact evaluation count (sizes of the probed lists), outside the timed window
        cells = _ref_probes(queries[idx], coarse, cfg["nprobe"])
        return float(np.asarray(sizes)[cells].sum())

    res = ref_run(evals_of, 1, 0, budget_s)
    what = "pqscan (the reference, baseline/_ref)" if kind == "reference" else "oracle/pqscan_oracle.py (port)"
    return {"value": res["value"], "unit": "evals/s", "cores": res["cores"], "kind": kind,
            "sample": f"{res['queries_per_step']} of {queries.shape[0]} queries, nprobe {cfg['nprobe']}, full index; "
                      f"{what}, fork pool x{res['cores']}; single-core median "
                      f"{res['single_core_ms_per_query']:.1f} ms/query"}


def make_ivf(args, ctx, dev):
    import paper_1712_02912_b200 as P
    from paper_1712_02912_b200 import datagen as G

    cfg = G.CONFIGS["cfg3"]
    books, coarse, sizes, codes, ids, queries = G.make_ivf_device(
        "cfg3", lambda b: P.DeviceQuantizer(P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], b), ctx),
        n=args.n_per_gpu, device=dev)
    return cfg, books, coarse, sizes, codes, ids, queries


def run_ivf(args):
    """cfg3 (IVFADC): the inverted lists are partitioned across the ranks
    (greedy by length); every rank holds the coarse quantizer,
    probes all 10k queries and scans its own lists; the per-rank top-100
    lists are all-gathered and merged (sharded.ShardedSearch.ivf).  The
    index and the query batch are fixed: strong scaling."""
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
    ctx.set_option(_lib.OPT_IVF_ENGINE, args.ivf_engine)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    t_build = time.perf_counter()
    cfg, books, coarse, sizes, codes, ids, queries = make_ivf(args, ctx, dev)
    pq = P.ProductQuantizer(cfg["m"], cfg["b"], cfg["d"], books)
    from paper_1712_02912_b200.sharded import ShardedSearch

    searcher = ShardedSearch.ivf(pq, coarse, sizes, codes, ids, rank, world, cfg["nprobe"], ctx=ctx)
    ivf = searcher.ivf_index
    n_total = int(codes.shape[0])
    host_index = None
    if not args.no_cpu_baseline and world == 1:
        host_index = (codes.cpu().numpy(), ids.cpu().numpy())
    del codes, ids
    torch.cuda.empty_cache()
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
        searcher.search(q_dev, r)
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
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" profiles the steps only
    for s in range(args.steps):
        flush.zero_()
        starts[s].record(stream)
        searcher.search(q_dev, r)
        ends[s].record(stream)
        scan_ns.append(ctx.stat(_lib.STAT_LAST_SCAN_NS))
        evals.append(ctx.stat(_lib.STAT_LAST_EVALS))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
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
        if world == 1:
            ivf.search(q_pin, ma, r, out=o_pin)
        else:
            d_, i_, c_ = searcher.search(torch.from_numpy(q_pin).to(dev, non_blocking=True), r)
            for dst, src in zip(o_pin, (d_, i_, c_)):
                torch.from_numpy(dst).copy_(src)
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
    engine = ctx.stat(_lib.STAT_LAST_SCAN_ENGINE)
    packed = engine == 6
    # list-major: every list's codes (+ V for the float scan, + the list's W table for the packed one) once
    hbm_alg = int(ivf_local_n(ivf)) * (m + (0 if packed else 4)) + (int(coarse.shape[0]) * m * 256 * 4 if packed else 0)
    lut_bound = (2.0 if packed else 1.0) * lut_peak
    hbm_peak = peaks.get("hbm_gbs", 6553.6)
    line = {
        "metric": metric_name("cfg3"), "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded stand-in for the BASELINE config, index built on the GPU; see DESIGN.md)",
        "config": {"workload": "IVFADC K=65536, residual PQ 8x8, nprobe 64", "baseline_config_index": 3,
                   "N_total": n_total, "N_per_gpu": int(ivf_local_n(ivf)), "queries": nq, "K": int(coarse.shape[0]),
                   "nprobe": ma, "m": m, "b": cfg["b"], "r": r, "d": cfg["d"],
                   "evals_per_step_per_gpu": evals_step,
                   "parallelism": f"inverted lists sharded x{world} (greedy by length)" if world > 1 else "single",
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
        "roofline": {"bound": "lut", "achieved": lut_rate, "peak": lut_bound, "unit": "Glookup/s",
                     "frac": lut_rate / lut_bound,
                     "traffic": _ncu_traffic("ivf_list8_kernel" if packed else "ivf_list_kernel"),
                     "traffic_note": _traffic_note(_ncu_entry("ivf_list8_kernel" if packed else "ivf_list_kernel")),
                     "kernel": ("ivf_list8_kernel (list-major, integer residual tables built per (list, 8 queries), two queries per word)"
                                if packed else "ivf_list_kernel (list-major, smem LUT)"),
                     "per_unit": f"{m} table lookups per probed (query, code); {evals_step:.3e} per launch",
                     "peak_source": (f"shared-memory wavefront rate {sm_count} SM x 64 lookups/clk (two queries per "
                                     f"32-bit word) x {f_mhz:.0f} MHz" if packed else
                                     f"shared-memory LUT rate {sm_count} SM x 32 lookups/clk x {f_mhz:.0f} MHz"),
                     "north_star_lut_frac": lut_rate / lut_peak,
                     "hbm": {"algorithmic_bytes": hbm_alg, "achieved_GBs": hbm_alg / (scan_ms / 1e3) / 1e9,
                             "peak_GBs": hbm_peak, "frac": hbm_alg / (scan_ms / 1e3) / 1e9 / hbm_peak},
                     "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step},
        "impl": "ours",
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_ivf(cfg, books, coarse.cpu().numpy(), sizes, host_index[0],
                                                host_index[1], queries, args.cpu_sample_s)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def ivf_local_n(ivf):
    return int(ivf.n)


def measured_i8_peak(seconds: float = 3.0):
    """tcgen05 kind::i8 peak of this GPU, measured live by tools/bin/pqs_peaks
    (tools/peaks.cu: M=128 N=256 K=32 MMAs back to back, operands resident):
    a burst figure and a sustained one (back-to-back launches for `seconds`).
    Falls back to the committed profiles/peaks_r02.json measurement."""
    exe = os.path.join(ROOT, "tools", "bin", "pqs_peaks")
    try:
        out = subprocess.run([exe, "i8", str(seconds)], capture_output=True, text=True, timeout=120)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        return {"burst": d["i8_mma"]["tops"], "sustained": d["i8_mma_sustained"]["tops"],
                "burst_mhz": d["i8_mma"]["sm_mhz"], "source": "measured live (tools/bin/pqs_peaks i8)"}
    except Exception as e:  # noqa: BLE001
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", "peaks_r02.json")))
            return {"burst": d["i8_mma"]["tops"], "sustained": d.get("i8_mma_sustained", d["i8_mma"])["tops"],
                    "burst_mhz": d["i8_mma"]["sm_mhz"],
                    "source": f"profiles/peaks_r02.json (committed measurement; live run failed: {e})"}
        except Exception:  # noqa: BLE001
            return None


def _ncu_entry(kernel: str):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(kernel)
    except (OSError, ValueError):
        return None


def _traffic_note(entry):
    """dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the kernel, from the committed ncu capture."""
    if not entry:
        return "no ncu capture committed for this kernel / config"
    return (f"DRAM read + write bytes of one launch, ncu --set full ({entry.get('capture')}): " + entry.get("note", "")).strip()


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
    ctx.set_option(_lib.OPT_SCAN8_ENGINE, args.scan8_engine)
    if args.tc_chunk_tiles:
        ctx.set_option(_lib.OPT_TC_CHUNK_TILES, args.tc_chunk_tiles)
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

    i8 = measured_i8_peak() if (rank == 0 and cfg["b"] == 4) else None
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
    if world == 1:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" profiles the steps only
        for s in range(args.steps):
            flush.zero_()
            starts[s].record(stream)
            step_device()
            ends[s].record(stream)
            scan_ns.append(ctx.stat(_lib.STAT_LAST_SCAN_NS))
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    else:
        # N > 1: the exchange + merge of step s overlaps the scan of step s+1
        # (ShardedSearch.search_stream); the K steps are timed as one region
        # (no per-step L2 flush: the 1 GB shard per GPU exceeds L2 anyway)
        starts[0].record(stream)
        for _ in searcher.search_stream((q_dev for _ in range(args.steps)), r):
            scan_ns.append(ctx.stat(_lib.STAT_LAST_SCAN_NS))
        ends[0].record(stream)
        for s in range(1, args.steps):
            starts[s], ends[s] = ends[0], ends[0]
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
        # tcgen05 kind::i8 one-hot GEMM: int8 MMA ops actually issued per launch,
        # against the microbenchmarked int8 MMA peak of this GPU: the sustained
        # figure when the timed region is a long one (> 1 s), else the burst one
        achieved = work / (scan_ms / 1e3) / 1e12
        regime = "sustained" if total_ms > 1000.0 else "burst"
        if i8 is not None:
            i8_peak = i8[regime]
            peak_source = (f"{i8['source']}: tcgen05.mma kind::i8 M=128 N=256 K=32 back to back, {regime} "
                           f"(burst {i8['burst']:.0f} / sustained {i8['sustained']:.0f} TOP/s)")
        else:
            i8_peak = 2.0 * peaks.get("bf16_tflops", 1660.1)
            peak_source = "fallback: 2 x MEASURED_PEAKS.json bf16_tflops (pqs_peaks unavailable)"
        roofline = {"bound": "tensor", "achieved": achieved, "peak": i8_peak, "unit": "TOP/s (int8)",
                    "frac": achieved / i8_peak,
                    "traffic": traffic_db.get("scan4tc_kernel_" + args.config, {}).get("bytes"),
                    "traffic_note": _traffic_note(traffic_db.get("scan4tc_kernel_" + args.config)),
                    "kernel": "scan4tc_kernel (tcgen05.mma kind::i8, M=128 N=256 K=256 per tile)",
                    "per_unit": "2 x 256 int8 MACs per (query, code) over 256-query groups and 128-code tiles "
                                f"({work:.3e} ops per launch)",
                    "peak_source": peak_source,
                    "lut_equivalent": lut, "hbm": hbm, "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step}
    elif engine == 5:
        # packed float filter: one 32-bit word carries two queries' entries, so a
        # conflict-free LDS.32 is 64 lookups per 128-byte wavefront: the bound is
        # the shared-memory wavefront rate (1 / clk / SM) x 64, twice the
        # north-star LUT rate (kept beside it)
        roofline = {"bound": "lut", "achieved": lut_rate, "peak": 2.0 * lut_peak, "unit": "Glookup/s",
                    "frac": lut_rate / (2.0 * lut_peak),
                    "per_unit": lut["per_unit"],
                    "peak_source": f"shared-memory wavefront rate {sm_count} SM x 1 wavefront/clk x 64 lookups "
                                   f"(two queries per 32-bit word) x {f_mhz:.0f} MHz",
                    "north_star_lut": lut,
                    "traffic": traffic_db.get("scan8p_kernel_" + args.config, {}).get("bytes"),
                    "traffic_note": _traffic_note(traffic_db.get("scan8p_kernel_" + args.config)),
                    "kernel": "scan8p_kernel (packed two-query words, PRMT-formed addresses, smem LUT)",
                    "hbm": hbm, "kernel_ms": scan_ms, "share_of_step": scan_ms / ms_per_step}
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
