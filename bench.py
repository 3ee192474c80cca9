#!/usr/bin/env python3
"""Benchmark: seconds per zeta function through the B200 controlled-reduction
engine (BASELINE.json metric), with the kernel roofline and the reference CPU
implementation timed beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config k3] [--impl ours|reference]

One step = one zeta function of the configured synthetic hypersurface
(reference generator rule: mt19937_64(seed), rng() % p per grevlex monomial,
smooth for both working sets).  `value` is the device-resident reduction
engine (seeds -> floor numerators for every Frobenius column, CUDA-event timed
on the engine stream); `e2e` is the whole zeta function through the public
C ABI (host coefficients in, Q out: setup, engine, final reduction, Frobenius
assembly, charpoly, Q recovery, point-count checks).  For N > 1 (torchrun),
Frobenius columns are partitioned across ranks, each rank reduces its columns
on its own GPU, and the per-rank column blocks are gathered over NCCL before
rank 0 recovers Q; times are the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seconds per zeta function (cubic fourfold p=7); mod-p^N reduction Gop/s vs roofline"

CONFIGS = {
    # name: (p, n, d, seed, description)
    "quintic": (7, 2, 5, 1, "smooth plane quintic curve /F7, seed 1 (configs[0])"),
    "k3": (11, 3, 4, 1, "random quartic K3 surface /F11, seed 1 (configs[1])"),
    "quintic_surface": (7, 3, 5, 1, "random quintic surface /F7, seed 1 (configs[2])"),
    "threefold": (13, 4, 3, 1, "random cubic threefold /F13, seed 1 (one of configs[3]'s batch)"),
    "fourfold": (7, 5, 3, 1, "random cubic fourfold /F7, seed 1 (configs[4])"),
    "fermat_fourfold_r1": (7, 5, 3, 0, "Fermat cubic fourfold /F7, reduced plan r_uniform=1"),
    # one step = the zeta functions of all 64 hypersurfaces; ranks take seeds
    # round-robin (replicas, no collective: SURVEY 8e)
    "threefold_batch": (13, 4, 3, 0, "batch of 64 random cubic threefolds /F13, seeds 0-63 (configs[3])"),
}
BATCH_SEEDS = 64


def merge_frobenius(frs):
    """sum the per-hypersurface counters of a batch step (ledger, kernel
    times, traffic, stage times); shape fields from the first"""
    out = dict(frs[0])
    for k in ("matvecs", "startups", "combines", "terms"):
        out[k] = sum(f[k] for f in frs)
    for sect in ("kernels", "traffic", "times"):
        out[sect] = {k: (sum(f[sect][k] for f in frs) if isinstance(v, (int, float)) else v)
                     for k, v in frs[0][sect].items()}
    return out


def hodge_counts(n, d):
    from math import comb
    h = []
    for m in range(1, n + 1):
        k = d * m - n - 1
        acc = 0
        j = 0
        while j * (d - 1) <= k and j <= n + 1:
            t = comb(n + 1, j) * comb(k - j * (d - 1) + n, n) if k - j * (d - 1) >= 0 else 0
            acc += -t if j & 1 else t
            j += 1
        h.append(acc if k >= 0 else 0)
    return h


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region"""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        if os.environ.get("DRZG_NO_CLOCKS"):  # diagnostics only: no sampling
            return self
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("DRZG_CLOCKS_MS", "250")],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def mark(self):
        """start of the timed region: waits until nvidia-smi is sampling
        (its start-up is over), then summary() keeps the samples after it"""
        t0 = time.time()
        while self.proc and time.time() - t0 < 15:
            try:
                if sum(1 for _ in open(self.path)) >= 2:
                    break
            except OSError:
                break
            time.sleep(0.05)
        try:
            self.f.flush()
            self.skip = sum(1 for _ in open(self.path))
        except (OSError, AttributeError):
            self.skip = 0

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        rows = []
        try:
            for ln, line in enumerate(open(self.path)):
                if ln < getattr(self, "skip", 0):
                    continue
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def committed_traffic(config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed `ncu --set full` capture of this config
    (profiles/r01/traffic_<config>.json, written from the .ncu-rep by hand;
    bench.py cannot run ncu itself), else null"""
    try:
        with open(os.path.join(ROOT, "profiles", "r01", f"traffic_{config}.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def int8_peak_tops(torch):
    """measured dense int8 tensor throughput (cuBLASLt via torch._int_mm)"""
    n = 8192
    a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda").t()
    best = 0.0
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return best


def reference_rate(cfg, coeffs, target_s=15.0):
    """reference run_policy on a bounded sample (oracle/_ref): matvecs per second
    with min(host cores, b) column threads, the reference's own parallelism"""
    from oracle import refapi
    p, n, d, _, _ = cfg
    h = hodge_counts(n, d)
    b = sum(h)
    threads = max(1, min(os.cpu_count() or 1, b))
    col = h[0] + (h[1] // 2 if len(h) > 1 and h[1] else 0)  # a middle-pole column
    per = 4
    while True:
        r = refapi.policy_sample(p, n, d, coeffs, col, per, threads)
        if r["seconds"] > target_s / 4 or per >= 4096:
            break
        per *= 4
    return r, threads, col, per


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    import paper_2602_24155_b200 as drzg
    p, n, d, seed, desc = cfg
    coeffs = drzg.random_hypersurface(p, n, d, seed=seed, fermat=(args.config.startswith("fermat")))
    total = json.load(open(os.path.join(ROOT, "profiles", f"ledger_{args.config}.json")))["matvecs"]
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        r, threads, col, per = reference_rate(cfg, coeffs, target_s=args.ref_seconds)
        proj = total * r["seconds"] / max(1, r["matvecs"])
        if i >= args.warmup:
            vals.append(proj)
        info = (r, threads, col, per)
    r, threads, col, per = info
    v = sum(vals) / len(vals)
    sample = (f"reference run_policy (p-chunk, lazy PEP) on column {col}'s top-pole seeds, {per} seeds x "
              f"{threads} threads ({r['matvecs']} matvecs in {r['seconds']:.2f} s), scaled by the exact "
              f"ledger of one zeta function ({total} matvecs)")
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64/u128 (reference)", "data": "synthetic",
            "config": {"workload": desc, "p": p, "n": n, "d": d},
            "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="k3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    p, n, d, seed, desc = cfg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import paper_2602_24155_b200 as drzg
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fermat = args.config.startswith("fermat")
    r_uniform = 1 if args.config.endswith("_r1") else 0
    coeffs = drzg.random_hypersurface(p, n, d, seed=seed, fermat=fermat)
    h = hodge_counts(n, d)
    b = sum(h)
    # columns partitioned across ranks (longest-processing-time by pole order)
    from paper_2602_24155_b200 import parallel
    all_cols = [parallel.partition_columns(n, d, world, r) for r in range(world)]
    mine = all_cols[rank] if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    batch = args.config == "threefold_batch"
    if batch:
        batch_coeffs = [drzg.random_hypersurface(p, n, d, seed=s) for s in range(rank, BATCH_SEEDS, world)]

    def step(profile=False):
        """one zeta function (or the rank's share of a batch); returns (device_s, json of this rank)"""
        if batch:
            zs = [drzg.zeta(p, n, d, co, device=local, profile=profile, verify_counts=True) for co in batch_coeffs]
            if not all(ok for z_ in zs for (_, _, ok) in z_["counts"]):
                raise RuntimeError("a point count disagrees with Q")
            fr_ = merge_frobenius([z_["frobenius"] for z_ in zs])
            z0 = dict(zs[0], seconds=sum(z_["seconds"] for z_ in zs))
            return fr_["kernels"]["device_ms"] / 1e3, z0, fr_
        if world == 1:
            z = drzg.zeta(p, n, d, coeffs, r_uniform=r_uniform, device=local, profile=profile,
                          verify_counts=True)
            return z["frobenius"]["kernels"]["device_ms"] / 1e3, z, z["frobenius"]
        fr = drzg.frobenius(p, n, d, coeffs, r_uniform=r_uniform, columns=mine, device=local, profile=profile)
        # one NCCL all_gather of the column blocks (62-bit limbs; see parallel.py)
        F = parallel.gather_frobenius(fr["F"], b, mine, world, all_cols, device=torch.device("cuda", local))
        z = drzg.charpoly(p, n, d, [str(x) for x in F], b, r_uniform=r_uniform) if rank == 0 else None
        return fr["kernels"]["device_ms"] / 1e3, z, fr

    dev_times, e2e_times, zeta_times, last = [], [], [], None
    # the sampler starts before the warm-up: nvidia-smi's start-up (NVML
    # init) stalls CUDA calls of this process for up to seconds, which must
    # not land in a timed step; it keeps sampling through the timed region
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev_s, z, fr = step()
            e1.record()
            torch.cuda.synchronize()
            e2e_s = e0.elapsed_time(e1) / 1e3
            if dist:
                tt = torch.tensor([dev_s, e2e_s], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dev_s, e2e_s = tt.tolist()
            dev_times.append(dev_s)
            e2e_times.append(e2e_s)
            if z and "seconds" in z:
                zeta_times.append(z["seconds"])
            last = (z, fr)
    if dist:
        dist.barrier()
    clocks = clk.summary()
    # profiled pass: per-kernel CUDA-event times on the engine stream
    _, _, frp = step(profile=True)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    z, fr = last
    value = sum(dev_times) / len(dev_times)
    e2e = sum(e2e_times) / len(e2e_times)
    kern = frp["kernels"]
    peak = int8_peak_tops(torch)
    ksum = kern["gemm_ms"] + kern["carry_ms"] + kern["gather_ms"] + kern["epilogue_ms"] + kern["other_ms"]
    # small systems (order <= 256) run the whole Dixon solve of a pole drop in
    # one launch (both products); larger ones launch the digit product and the
    # block-sparse carry product separately
    fused = kern["carry_launches"] == 0 and kern.get("carry_macs", 0) > 0
    gemm_macs = kern["gemm_macs"] + (kern["carry_macs"] if fused else 0)
    gemm_avg_ms = kern["gemm_ms"] / max(1, kern["gemm_launches"])
    achieved = 2 * gemm_macs / max(1e-9, kern["gemm_ms"] / 1e3) / 1e12
    carry = None
    if not fused:
        carry_tops = 2 * kern.get("carry_macs", 0) / max(1e-9, kern["carry_ms"] / 1e3) / 1e12
        carry = {"kernel": "tc::gemm_kernel (block-sparse carry product + residual epilogue)",
                 "achieved_tops": carry_tops, "frac": carry_tops / peak if peak else None,
                 "share_of_kernel_time": kern["carry_ms"] / ksum if ksum else None}
    if not fused:
        kname = "tc::gemm_kernel (digit product y_k = bal(Cq . in_k))"
    elif fr["nL"] <= 256:
        kname = "tc::dixon_fused_kernel (digit + carry products of every digit, one launch per pole drop)"
    else:
        kname = "tc::dixon_flow_kernel (dense digit + block-sparse carry tiles of every digit, one dataflow launch)"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    total_matvecs = fr["matvecs"] if world == 1 else None
    if world == 1:
        with open(os.path.join(ROOT, "gpurun_out", f"ledger_{args.config}.json"), "w") as f:
            json.dump({"matvecs": fr["matvecs"], "startups": fr["startups"], "combines": fr["combines"]}, f)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            r, threads, col, per = reference_rate(cfg, coeffs, target_s=args.ref_seconds)
            proj = fr["matvecs"] * r["seconds"] / max(1, r["matvecs"])
            cpu = {"value": proj, "unit": "s", "cores": threads, "kind": "reference",
                   "sample": (f"reference run_policy (p-chunk, lazy PEP) on column {col}'s top-pole seeds, "
                              f"{per} seeds x {threads} threads: {r['matvecs']} matvecs in {r['seconds']:.2f} s; "
                              f"scaled by this zeta function's exact ledger ({fr['matvecs']} matvecs, "
                              f"identical to the reference's)")}
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": "s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    # mod-p^N reduction Gop/s = 2 side^2 per matvec x matvecs / s
    gops = 2.0 * fr["side"] ** 2 * fr["matvecs"] / value / 1e9 if world == 1 else None
    traffic = committed_traffic(args.config)
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "i8", "data": "synthetic",
        "config": {"workload": desc, "p": p, "n": n, "d": d, "M": fr["M"], "digits": fr["digits"],
                   "side": fr["side"], "nL": fr["nL"], "b": b, "parallelism": f"columns/{world}",
                   "l2": "flushed between steps (256 MiB write)", "policy": "p-chunk"},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": fr["traffic"]["h2d_bytes"] + 8 * len(coeffs),
                "d2h_bytes_per_step": fr["traffic"]["d2h_bytes"]},
        "gpu_launches": fr["traffic"]["launches"] * args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
                     "frac": achieved / peak if peak else None, "traffic": (traffic or {}).get("bytes_per_launch"),
                     "traffic_source": (traffic or {}).get("source"),
                     "kernel": kname, "avg_launch_ms": gemm_avg_ms,
                     "share_of_kernel_time": kern["gemm_ms"] / ksum if ksum else None,
                     "peak_source": "measured on this box: torch._int_mm 8192^3 int8 (cuBLASLt), best of 5"},
        "reduction_gops": gops,
        "carry_gemm": carry,
        "ledger": {"matvecs": fr["matvecs"], "startups": fr["startups"], "combines": fr["combines"],
                   "terms": fr["terms"]},
        "per_step_s": {"device": [round(x, 4) for x in dev_times], "e2e": [round(x, 4) for x in e2e_times],
                       "zeta_call": [round(x, 4) for x in zeta_times]},
        "stage_seconds": fr["times"], "kernels_ms": kern,
        "cpu_baseline": cpu, "clocks": clocks,
        "Q_head": (z["Q"][:4] if z and "Q" in z else (z["candidates"][0][:4] if z else None)),
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
