"""bench.py — the OEM hot path on B200: Gram fp64 TFLOP/s and full-path fit seconds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl oem|reference]

For N > 1 the driver launches one process per GPU with torch.distributed.run; X is row-sharded
(rank r owns global rows [r n/N, (r+1) n/N), generated in place on its GPU) and the raw Gram is
combined with one NCCL allreduce inside oem_gram; n is fixed as N grows
("scaling": "strong"). One step = the whole hot path over the workload: a2 Gram pass
(+ a5 combine) -> a6 normalise -> a7 d -> a8 lambda grid -> a9/a10 the OEM paths for every
penalty. `value` = whole-job Gram TFLOP/s (algorithmic n p (p+3) flops, all ranks, over the max
over ranks of the Gram-phase device time); `fit_seconds` = device time of the whole step.
Inputs (80 GB for cfg4) are far larger than the 126 MB L2, so no flush is needed.

The reference arm (--impl reference) is the repo's CPU oracle (oracle/), timed as it stands on
the host cores on a bounded row sample of the same workload: this run has no reference
implementation to install (the reference is a paper), see DESIGN.md §8.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen as dg  # noqa: E402
from datagen.configs import CONFIGS, groups_of  # noqa: E402

METRIC = "Gram fp64 TFLOP/s (X^TX+X^Ty) and full-path fit seconds at 1/2/4/8 B200"
FP64_PEAK_TFLOPS = 37.06   # measured DMMA peak, profiles/fp64_peak_r01.log (MEASURED_PEAKS.json has no fp64)
HBM_PEAK_GBS = 6549.8      # MEASURED_PEAKS.json (copy bandwidth, burst)


def gram_flops(n, p):
    """Algorithmic flops of the Gram pass: n p (p+1) (SYRK upper + diagonal) + 2 n p (X^T y)."""
    return float(n) * p * (p + 3)


def weighted_flops(n, p):
    """Algorithmic flops of one weighted pass: n p (p+1) (SYRK) + 2 n p (X^T W z)
    + 2 n p (eta = X beta) + n p (weight scaling) = n p (p+6)."""
    return float(n) * p * (p + 6)


def sample_flops(cfg, X):
    """Algorithmic flops of the Gram pass over the sample rows X: dense n p (p+3); for the sparse
    workload (f4) the products of each row's nonzeros, m (m+1) + 4 m + 2 per row (R#38)."""
    if cfg.spec.design == dg.DG_SPARSE:
        m = (X != 0).sum(axis=1).astype(float)
        return float(np.sum(m * (m + 1) + 4 * m + 2))
    return gram_flops(X.shape[0], X.shape[1])


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([s.strip() for s in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, budget_s=15.0, path_inputs=None):
    """The oracle's Gram (oracle/oracle.c, compensated fp64, all host cores) on a bounded row
    sample of the workload; rows come from the host generator (untimed). With path_inputs (the
    full-data raw Gram, X^T y, n, d and grid from the GPU step, linear non-fold workloads) the
    oracle's path solve (O6, single thread) is timed on the same problem, when its estimated cost
    fits the budget, and an oracle fit-seconds estimate is reported."""
    import oracle as orc
    cores = os.cpu_count() or 1
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    probe = max(64, min(2000, int(2e8 / (cfg.p * cfg.p))))
    X, y = dg.rows_host(cfg.spec, bt, 0, probe)
    t0 = time.perf_counter()
    orc.gram(X, y, nthreads=cores)
    dt = time.perf_counter() - t0
    rows = int(min(cfg.n, max(probe, probe * budget_s / max(dt, 1e-6))))
    rows = min(rows, probe * 64)
    X, y = dg.rows_host(cfg.spec, bt, 0, rows)
    t0 = time.perf_counter()
    orc.gram(X, y, nthreads=cores)
    dt = time.perf_counter() - t0
    out = {"value": sample_flops(cfg, X) / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
           "cpu_model": cpu_model(),
           "sample": f"oracle Gram (compensated fp64, {cores} threads) over rows 0..{rows} of {cfg.name} "
                     f"(n={cfg.n}, p={cfg.p}), {dt:.2f} s"}
    if path_inputs is not None:
        G, c, n, d, lams, grp, ngroups, est = path_inputs
        if est <= 4 * budget_s:
            t0 = time.perf_counter()
            for q, (fam, gamma, alpha) in enumerate(cfg.penalties):
                g = grp if fam.startswith("grp") or fam == "sgl" else None
                orc.oem_path(G / n, c / n, d, fam, lams[q], gamma, alpha, group=g,
                             ngroups=ngroups if g is not None else 0)
            tp = time.perf_counter() - t0
            gram_s = dt * cfg.n / rows
            out["path_seconds"] = tp
            out["fit_seconds_est"] = gram_s + tp
            out["sample"] += f"; oracle path solve (1 thread) of the full problem {tp:.1f} s; fit estimate = " \
                             f"Gram extrapolated to n + path"
    return out


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as orc
    cores = os.cpu_count() or 1
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    rows = max(256, int(3e9 / (cfg.p * (cfg.p + 3))))  # a few seconds of oracle work per step
    X, y = dg.rows_host(cfg.spec, bt, 0, rows)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        G, c, yy = orc.gram(X, y, nthreads=cores)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    v = sample_flops(cfg, X) / (sum(times) / len(times)) / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox generator, DESIGN.md §4)",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "penalties": [f for f, _, _ in cfg.penalties],
                       "nlambda": cfg.nlambda, "folds": cfg.folds, "logistic": cfg.logistic,
                       "parallelism": f"CPU oracle on {cores} host threads (no GPU)", "sample_rows": rows},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": f"oracle Gram over rows 0..{rows} of {cfg.name} per step"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ multi-GPU validation
def validate_combine(cfg, ctx, Xd, yd, r0, res, rank, world, dist, torch, csr=None):
    """Untimed checks of the row-sharded combine at N > 1: (1) the SHA-256 of each rank's combined
    statistics and coefficient paths, all-gathered: they must be identical on every rank (NCCL
    Ring/Simple gives every rank the same reduced bits; the path solve is a deterministic replica);
    (2) on rank 0, the combined Gram on 8 columns (the first 4 and 4 in the last 128-column
    panel) against the oracle's compensated sums over all n rows (host generator, those columns)."""
    import hashlib

    from paper_1801_09661_b200 import oem_gram, oem_gram_csr, oem_gram_folds
    if csr is not None:
        G, c, yy, _ = oem_gram_csr(ctx, *csr, cfg.p)
        stats = (G, c, yy)
    elif cfg.folds:
        Gk, ck, yyk, cnt = oem_gram_folds(ctx, Xd, yd, cfg.folds, row_offset=r0)
        G, c, yy = Gk.sum(0), ck.sum(0), yyk.sum()
        stats = (Gk, ck, yyk)
    else:
        G, c, yy, _ = oem_gram(ctx, Xd, yd)
        stats = (G, c, yy)
    h = hashlib.sha256()
    for t in stats + (res.beta, res.d):
        h.update(t.detach().cpu().numpy().tobytes())
    mine = h.hexdigest()
    digests = [None] * world
    if world > 1:
        dist.all_gather_object(digests, mine)
    else:
        digests = [mine]
    out = {"digests_equal": len(set(digests)) == 1, "digest": mine[:16]}
    if rank == 0:
        import oracle as orc
        p = cfg.p
        # block-equicorrelated columns are generated independently (first 4 + last 4 columns, two
        # panels, and y from the active groups); AR(1) columns need every earlier column and y
        # every support column, so those designs check the first 8 columns of G only
        block = cfg.spec.design in (dg.DG_BLOCK, dg.DG_SPARSE)   # independent columns
        blocks = [(0, 4), (p - 4, 4)] if block and p > 8 else [(0, min(8, p))]
        idx = np.concatenate([np.arange(a, a + m) for a, m in blocks])
        bt = dg.beta(cfg.spec, cfg.explicit_beta)
        acc = orc.GramAccumulator(idx.size)
        chunk = 1_000_000
        for r in range(0, cfg.n, chunk):
            nr = min(chunk, cfg.n - r)
            parts, y = [], None
            for a, m in blocks:
                X, yb = dg.rows_host(cfg.spec, bt, r, nr, a, m, want_y=block and y is None)
                parts.append(X)
                y = yb if y is None else y
            acc.add(np.ascontiguousarray(np.hstack(parts)), y if block else np.zeros(nr))
        Go, co, yyo = acc.result()
        Gh = G.cpu().numpy()[np.ix_(idx, idx)]
        dd = np.sqrt(np.outer(np.diag(Go), np.diag(Go)))
        gerr = float(np.max(np.abs(Gh - Go) / dd))
        out.update({"oracle_columns": idx.tolist(), "gram_scale_err": gerr})
        out["oracle_ok"] = gerr <= 1e-12
        if block:
            cerr = float(np.max(np.abs(c.cpu().numpy()[idx] - co) / np.sqrt(np.diag(Go) * yyo)))
            out.update({"xty_scale_err": cerr, "yty_rel_err": abs(float(yy) - yyo) / yyo})
            out["oracle_ok"] = out["oracle_ok"] and cerr <= 1e-12 and out["yty_rel_err"] <= 1e-12
    ok = torch.tensor([1.0 if out["digests_equal"] and out.get("oracle_ok", True) else 0.0],
                      dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    out["ok"] = bool(ok.item() == 1.0)
    return out


# ------------------------------------------------------------------ the GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="oem", choices=["oem", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--validate", action="store_true",
                    help="run the multi-GPU validation (digests + oracle column sample) also at N = 1")
    ap.add_argument("--n", type=int, default=0, help="override n (development only; not a bench number)")
    args = ap.parse_args()
    cfg = CONFIGS[args.workload]
    if args.n:
        cfg = cfg.with_n(args.n)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_1801_09661_b200 import Context, oem, oem_fit_path, oem_gram, oem_gram_csr, oem_gram_folds
    from paper_1801_09661_b200.oem import oem_fit_logistic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        # a fixed NCCL algorithm / protocol: bitwise-reproducible combines
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [oem.oem_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = Context(local, world, rank, obj[0])
    else:
        ctx = Context(local)

    def barrier():
        if world > 1:
            dist.barrier()

    def sum_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    # ---- a1: this rank's rows, generated in place on its GPU (untimed)
    n, p = cfg.n, cfg.p
    r0, r1 = rank * n // world, (rank + 1) * n // world
    nl = r1 - r0
    bt = dg.beta(cfg.spec, cfg.explicit_beta)
    ldx = p + (p & 1)
    sparse = cfg.spec.design == dg.DG_SPARSE
    csr = None
    if sparse:
        # f4: this rank's rows in CSR form (row offsets, ascending column indices, values)
        csr = dg.csr_cuda(cfg.spec, bt, r0, nl)
        Xs = Xd = None
        yd = csr[3]
        m = (csr[0][1:] - csr[0][:-1]).double()
        # algorithmic work of the sparse pass: row i has m_i nonzeros and contributes
        # m_i (m_i + 1)/2 + m_i + 1 products (2 flops each); it reads row_ptr, y and 12 B per nonzero
        sp_flops_local = float((m * (m + 1) + 4 * m + 2).sum())
        sp_bytes_local = float(8 * (nl + 1) + 8 * nl + 12 * int(csr[1].numel()))
        sp_nnz = int(csr[1].numel())
    else:
        Xs = torch.empty((nl, ldx), dtype=torch.float64, device="cuda")
        Xd = Xs[:, :p]
        yd = torch.empty(nl, dtype=torch.float64, device="cuda")
        btd = torch.from_numpy(bt).cuda()
        dg.rows_cuda(cfg.spec, btd.data_ptr(), r0, nl, Xs.data_ptr(), ldx, yd.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    grp = groups_of(cfg)
    ngroups = p // cfg.group_size if grp is not None else 0

    def step(X, y):
        """One pass of the whole hot path; returns the fit result (device tensors)."""
        if cfg.logistic:
            return oem_fit_logistic(ctx, X, y, cfg.penalties[0], nlambda=cfg.nlambda)
        if cfg.folds:
            G, c, yy, cnt = oem_gram_folds(ctx, X, y, cfg.folds, row_offset=r0)
        else:
            G, c, yy, nn = oem_gram_csr(ctx, *csr[:3], y, p) if sparse else oem_gram(ctx, X, y)
            cnt = [nn]
        return oem_fit_path(ctx, G, c, cnt, cfg.penalties, nlambda=cfg.nlambda, fold_mode=bool(cfg.folds),
                            group=grp, ngroups=ngroups)

    for _ in range(args.warmup):
        res = step(Xd, yd)
    torch.cuda.synchronize()
    oem.set_timing(ctx, True)
    oem.stats(ctx, reset=True)
    clocks = Clocks(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record()
    for k in range(args.steps):
        res = step(Xd, yd)
        ev[k + 1].record()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = ev[0], ev[-1]
    step_times = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    clk = clocks.stop()
    st = oem.stats(ctx, reset=True)
    oem.set_timing(ctx, False)
    total_ms = e0.elapsed_time(e1)
    gram_phase_ms = st["gram_ms"] + st["reduce_ms"] + st["allreduce_ms"]
    step_ms = max_over_ranks(total_ms / args.steps)
    step_median_ms = max_over_ranks(statistics.median(step_times))
    step_min_ms = max_over_ranks(min(step_times))
    gram_step_ms = max_over_ranks(gram_phase_ms / args.steps)
    kernel_ms = max_over_ranks(st["gram_ms"] / args.steps)
    path_step_ms = max_over_ranks((st["power_ms"] + st["path_ms"]) / args.steps)  # every rank calls (collective)
    power_step_ms = max_over_ranks(st["power_ms"] / args.steps)                    # a7 (the d rule) alone
    passes = 1
    if cfg.logistic:
        passes = max(1, round(st["launches"] / max(1, args.steps)))  # informational only
    flops_step = gram_flops(n, p)
    if cfg.logistic:
        # every outer step is one weighted pass; count them from the fit
        outer = sum(res.outer_iters)
        flops_step = weighted_flops(n, p) * outer
    if sparse:
        flops_step = max_over_ranks(sp_flops_local) if world == 1 else sum_over_ranks(sp_flops_local)
    value = flops_step / (gram_step_ms * 1e-3) / 1e12
    # roofline of the dominant kernel (the tensor-core Gram kernel): algorithmic flops per
    # launch over its event-timed launch duration on this rank
    per_launch_flops = (weighted_flops(nl, p) * sum(res.outer_iters)) if cfg.logistic else gram_flops(nl, p)
    achieved = per_launch_flops / (st["gram_ms"] / args.steps * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")   # one `ncu --set full` capture per kernel
    if os.path.exists(prof):
        try:
            key = "sparse" if sparse else f"gram_{cfg.name}"
            traffic = json.load(open(prof)).get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if sparse:
        # the sparse pass is bound by reading the CSR arrays: algorithmic bytes per launch
        # (8 (n+1) row offsets + 8 n for y + 12 per nonzero) over the event-timed launch
        achieved = sp_bytes_local / (st["gram_ms"] / args.steps * 1e-3) / 1e9
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "kernel": "oem::gram_kernel (TMA + DMMA.8x8x4)",
                "peak_source": "measured FP64 DMMA microbenchmark (profiles/fp64_peak_r01.log); "
                               "MEASURED_PEAKS.json carries no fp64 figure",
                "share_of_step": st["gram_ms"] / max(total_ms, 1e-9),
                "hbm_gbs": 8.0 * nl * (p + 1) * (sum(res.outer_iters) if cfg.logistic else 1)
                           / (st["gram_ms"] / args.steps * 1e-3) / 1e9}
    if sparse:
        roofline.update({"bound": "hbm", "peak": HBM_PEAK_GBS, "unit": "GB/s", "frac": achieved / HBM_PEAK_GBS,
                         "kernel": "oem::sparse_gram_kernel (CSR, cp.async ring, warp-owned triangle rows)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                         "hbm_gbs": achieved, "bytes_per_launch": sp_bytes_local, "nnz_local": sp_nnz})
    launches = int(st["launches"])

    # ---- e2e: the same metric through the public API with HOST buffers (pinned). Linear
    # workloads stream X, y from host memory through the Gram kernel (oem_gram_host /
    # oem_gram_folds_host, f4: copies overlapped with the contraction); the logistic workload
    # copies X, y once per step (its weighted pass re-reads X every outer step). The D2H of the
    # coefficient paths is inside the timed step.
    e2e = None
    if args.e2e_steps > 0:
        try:
            from paper_1801_09661_b200 import oem_gram_folds_host, oem_gram_host
            if sparse:   # pinned host copies of the CSR arrays; copied to the device inside each step
                hcsr = [t.cpu().pin_memory() for t in csr]
                in_bytes = sum(t.numel() * t.element_size() for t in hcsr)
            else:
                Xh = torch.empty((nl, ldx), dtype=torch.float64, pin_memory=True)
                yh = torch.empty(nl, dtype=torch.float64, pin_memory=True)
                Xh.copy_(Xs)
                yh.copy_(yd)
                in_bytes = nl * ldx * 8 + nl * 8
            torch.cuda.synchronize()
            blk = 1 << 20
            out_bytes = 0
            gram_ms = 0.0
            barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t2 = torch.cuda.Event(enable_timing=True)
            for it in range(args.e2e_steps + 1):   # iteration 0: untimed warm-up (staging buffers, plans)
                if it == 1:
                    torch.cuda.synchronize()
                    barrier()
                    gram_ms = 0.0
                    t0.record()
                ta = torch.cuda.Event(enable_timing=True)
                tb = torch.cuda.Event(enable_timing=True)
                ta.record()
                if cfg.logistic:
                    Xs.copy_(Xh, non_blocking=True)
                    yd.copy_(yh, non_blocking=True)
                    r = oem_fit_logistic(ctx, Xd, yd, cfg.penalties[0], nlambda=cfg.nlambda)
                    tb.record()
                elif sparse:
                    for dst, src in zip(csr, hcsr):
                        dst.copy_(src, non_blocking=True)
                    G, c, yy, nn = oem_gram_csr(ctx, *csr[:3], csr[3], p)
                    tb.record()
                    r = oem_fit_path(ctx, G, c, [nn], cfg.penalties, nlambda=cfg.nlambda, group=grp, ngroups=ngroups)
                else:
                    if cfg.folds:
                        G, c, yy, cnt = oem_gram_folds_host(ctx, Xh[:, :p], yh, cfg.folds, row_offset=r0, block_rows=blk)
                    else:
                        G, c, yy, nn = oem_gram_host(ctx, Xh[:, :p], yh, block_rows=blk)
                        cnt = [nn]
                    tb.record()
                    r = oem_fit_path(ctx, G, c, cnt, cfg.penalties, nlambda=cfg.nlambda, fold_mode=bool(cfg.folds),
                                     group=grp, ngroups=ngroups)
                hb = r.beta.cpu()
                out_bytes = hb.numel() * 8
                torch.cuda.synchronize()
                gram_ms += ta.elapsed_time(tb)
            t2.record()
            torch.cuda.synchronize()
            barrier()
            e2e_step_ms = max_over_ranks(t0.elapsed_time(t2) / args.e2e_steps)
            e2e_gram_ms = max_over_ranks(gram_ms / args.e2e_steps)
            if cfg.logistic:
                e2e_val = flops_step / (e2e_step_ms * 1e-3) / 1e12
                note = ("logistic: H2D of X, y (pinned) once per step + the whole proximal-Newton fit; value = "
                        "weighted-Gram flops over the whole step")
            elif sparse:
                e2e_val = flops_step / (e2e_gram_ms * 1e-3) / 1e12
                note = ("sparse: H2D of the pinned CSR arrays and y + the CSR Gram pass (the Gram phase); "
                        "fit_seconds adds the path solve and the D2H of the paths")
            else:
                e2e_val = flops_step / (e2e_gram_ms * 1e-3) / 1e12
                note = ("Gram phase streamed from pinned host memory in 2^20-row blocks (oem_gram_host, copies "
                        "overlapped with the kernel); fit_seconds adds the path solve and the D2H of the paths")
            e2e = {"value": e2e_val, "unit": "TFLOP/s",
                   "h2d_bytes_per_step": int(in_bytes) * world,
                   "d2h_bytes_per_step": int(out_bytes) * world,
                   "fit_seconds": e2e_step_ms / 1e3, "gram_phase_ms": e2e_gram_ms,
                   "h2d_gbs": in_bytes / (e2e_gram_ms * 1e-3) / 1e9 if not cfg.logistic else None,
                   "note": note}
        except Exception as ex:  # pinned memory exhausted etc.: report, do not fake
            e2e = {"value": None, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "error": repr(ex)[:200]}

    # ---- multi-GPU self-validation (untimed): every rank must hold bitwise-identical combined
    # statistics and fits (all-gathered digests), and rank 0 checks the combined Gram against the
    # oracle on a column sample over ALL n rows
    validation = None
    if (world > 1 or args.validate) and not cfg.logistic:
        validation = validate_combine(cfg, ctx, Xd, yd, r0, res, rank, world, dist, torch, csr)
        if not validation["ok"]:
            if rank == 0:
                print(json.dumps({"error": "multi-GPU validation failed", "validation": validation}), flush=True)
            ctx.close()
            if world > 1:
                dist.destroy_process_group()
            return 1

    pin = None
    if not args.no_cpu_baseline and not cfg.logistic and not cfg.folds:
        Gf, cf, _, nf = oem_gram_csr(ctx, *csr, p) if sparse else oem_gram(ctx, Xd, yd)   # every rank: a collective
        iters = int(res.iters.sum())
        est = iters * float(p) * p / 2e9  # ~2 GFLOP/s single-thread naive loops
        pin = (Gf.cpu().numpy(), cf.cpu().numpy(), nf, float(res.d[0]),
               [res.lam[0, q].cpu().numpy() for q in range(len(cfg.penalties))], grp, ngroups, est)
    barrier()
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, path_inputs=pin)
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "fit_seconds": step_ms / 1e3,
            "step_ms_median": step_median_ms, "step_ms_min": step_min_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox4x32-10 generator, generated in place on each GPU)",
            "config": {"workload": cfg.name, "n": n, "p": p, "penalties": [f for f, _, _ in cfg.penalties],
                       "nlambda": cfg.nlambda, "folds": cfg.folds, "logistic": cfg.logistic,
                       "parallelism": f"rows sharded over {world} GPU(s), NCCL allreduce of the packed Gram",
                       "l2": "inputs larger than L2 (no flush needed)",
                       "step": "Gram pass (+allreduce) -> normalise -> d -> lambda grid -> OEM paths"},
            "gram_phase_ms": gram_step_ms, "gram_kernel_ms": kernel_ms,
            "path_phase_ms": path_step_ms,
            "iters": int(res.iters.sum()) if not cfg.logistic else int(sum(res.inner_iters)),
            "path_us_per_iter": (None if cfg.logistic else
                                 1e3 * path_step_ms / max(1, int(res.iters.sum(-1).max()))),
            "roofline": roofline, "clocks": clk, "gpu_launches": launches, "e2e": e2e,
            "nccl": {"version": ".".join(str(v) for v in torch.cuda.nccl.version()) if world > 1 else None,
                     "algo": os.environ.get("NCCL_ALGO"), "proto": os.environ.get("NCCL_PROTO")},
            "cpu_baseline": cpu,
            "power_ms": power_step_ms,
            "validation": validation,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
