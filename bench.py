#!/usr/bin/env python3
"""Benchmark: seconds per zeta function through the B200 controlled-reduction
engine (BASELINE.json metric), with the kernel roofline and the reference CPU
implementation timed beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config k3] [--impl ours|reference]

One step = one zeta function of the configured synthetic hypersurface
(reference generator rule: mt19937_64(seed), rng() % p per grevlex monomial,
smooth for both working sets), through the public C ABI (drzg_zeta): setup,
seeds, the device engine, the final reduction, Frobenius assembly, charpoly,
Q recovery and the point-count checks.
  value  the zeta call's own wall time (run_zeta, zeta.hpp:438-549), every stage
  e2e    the same call timed from Python with CUDA events around it: host
         coefficients in, JSON (Q) out; h2d/d2h count every byte it copies
For N > 1 (torchrun), Frobenius columns are partitioned across ranks, each
rank reduces its columns on its own GPU, the column blocks are gathered over
NCCL, and rank 0 runs run_zeta's battery on the gathered F (drzg_zeta_from_F);
times are the max over ranks.

The default config is the K3 surface (configs[1]): the metric's cubic
fourfold (configs[4]) takes minutes per zeta function on one B200, so 5 + 20
of them do not fit the driver's run.  At N = 1 the default run therefore also
times ONE complete fourfold zeta function (key "fourfold": warm-up on one
column, then the whole zeta function with both point-count checks, clocks,
ledger against the reference's replayed ledger, Q hash, per-kernel roofline).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seconds per zeta function (cubic fourfold p=7); mod-p^N reduction Gop/s vs roofline"
GOLD = os.path.join(ROOT, "tests", "golden")

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
BATCH_WORKERS = 8  # concurrent zeta functions per rank (scripts/batch_ab.py: 26.1 s at 1, 16.7 s at 8)
# the reference's full ledger of each config (tests/golden: real reference
# runs; ledger_replay_*: the reference's value-free replay, which equals the
# real ledger on every fixture -- tests/test_oracle.py)
LEDGER_SOURCE = {"quintic": "quintic_f7_s1.json", "k3": "k3_f11_s1.json", "threefold": "threefold_f13_s1.json",
                 "fourfold": "ledger_replay_fourfold.json", "quintic_surface": "ledger_replay_quintic_surface.json"}
# series truncation of the reference's bounded sample (same hypersurface, same
# limb count, every column and pole; scaled by the ledger ratio)
SAMPLE_NM = {"k3": 4, "threefold": 4}
FOURFOLD_COUNT_BUDGET = 1_000_000_000  # both count checks: #P^5(F_49) = 2.9e8 points


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

    def __init__(self, index, tag=""):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}{tag}.csv")

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
    (profiles/<round>/traffic_<config>.json, written from the .ncu-rep by hand;
    bench.py cannot run ncu itself), else null"""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, f"traffic_{config}.json")) as f:
                return json.load(f)
        except (OSError, ValueError):
            continue
    return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


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


# --------------------------------------------------------------------------
# the reference on the host cores (oracle/_ref: the UNMODIFIED reference
# headers compiled in place).  Nothing here imports the product package.

def full_ledger(config):
    name = LEDGER_SOURCE.get(config)
    if not name:
        return None
    try:
        with open(os.path.join(GOLD, name)) as f:
            g = json.load(f)
    except OSError:
        return None
    return dict(g["ledger"], source=f"tests/golden/{name}")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_measure(config, coeffs, threads):
    """one timed reference run on the host cores: the whole zeta function when
    it fits a bench step (quintic), else frobenius_matrix at a series-truncated
    plan (N_m = SAMPLE_NM: every column and pole, the same limb count, so the
    same per-matvec cost) scaled by the ratio of the exact ledgers; for the
    fourfold (two limbs, beyond the reference here) one reference linrec_eval
    step at its size (p=7, M=24, side 3003) times the replayed ledger."""
    from oracle import refapi
    p, n, d, seed, _ = CONFIGS[config]
    full = full_ledger(config)
    if config == "quintic":
        t0 = time.time()
        z = refapi.zeta(p, n, d, coeffs, threads=threads)
        secs = time.time() - t0
        return {"value": secs, "kind": "reference", "projection": False,
                "sample": f"the whole reference run_zeta (p-chunk, lazy PEP, {threads} column threads): "
                          f"{z['matvecs']} matvecs, Q head {z['Q'][:3]}"}
    if config in SAMPLE_NM and full:
        nm = SAMPLE_NM[config]
        t0 = time.time()
        fr = refapi.frobenius(p, n, d, coeffs, threads=threads, nm=nm)
        secs = time.time() - t0
        proj = secs * full["matvecs"] / max(1, fr["matvecs"])
        return {"value": proj, "kind": "reference", "projection": True,
                "sample": (f"reference frobenius_matrix (p-chunk, lazy PEP, {threads} column threads) of the same "
                           f"hypersurface at N_m={nm} (M={fr['plan']['M']}, every column and pole): "
                           f"{fr['matvecs']} matvecs in {secs:.2f} s, scaled to the full ledger "
                           f"({full['matvecs']} matvecs, {full['source']})"),
                "sample_seconds": secs}
    if config == "fourfold" and full:
        import numpy as np
        rng = np.random.default_rng(7)
        side, beta = 3003, 7 ** 12
        A = rng.integers(0, beta, size=2 * side * side, dtype=np.uint64)
        B = rng.integers(0, beta, size=2 * side * side, dtype=np.uint64)
        w = rng.integers(0, beta, size=2 * side, dtype=np.uint64)
        t0 = time.time()
        refapi.linrec_eval(7, 24, side, A, B, 0, w)
        step = time.time() - t0
        proj = step * full["matvecs"] / max(1, min(threads, 22))
        return {"value": proj, "kind": "reference", "projection": True,
                "sample": (f"one reference linrec_eval step at the fourfold's size (p=7, M=24: 2 limbs, side 3003, "
                           f"generic path) took {step:.2f} s on one core; x {full['matvecs']} matvecs "
                           f"({full['source']}) / min(cores, 22 columns); excludes the reference's per-column "
                           f"RuvContext and ~150 GB of seed vectors, so a lower bound"),
                "sample_seconds": step}
    return None


def validation():
    """the projection method checked against complete reference runs in the
    dev container (profiles/r02/cpu_baseline_validation.json)"""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "cpu_baseline_validation.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def run_reference(args, cfg, rank):
    """--impl reference: the reference's own CPU implementation on the host
    cores (oracle/_ref), same config/metric/unit; rank 0 only"""
    if rank != 0:
        return
    from oracle import refapi
    p, n, d, seed, desc = cfg
    if args.config in ("threefold_batch", "fermat_fourfold_r1"):
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": f"no reference arm for config {args.config}"}))
        return
    coeffs = [int(x) for x in refapi.hypersurface(p, n, d, seed=seed)]
    threads = host_threads()
    vals, info = [], None
    for i in range(args.warmup + args.steps):
        info = reference_measure(args.config, coeffs, threads)
        if info is None:
            print(json.dumps({"impl": "reference", "metric": METRIC, "unavailable": "no reference ledger"}))
            return
        if i >= args.warmup:
            vals.append(info["value"])
    v = sum(vals) / len(vals)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64/u128 (reference)", "data": "synthetic",
            "config": {"workload": desc, "p": p, "n": n, "d": d},
            "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": info["kind"],
                             "projection": info["projection"], "sample": info["sample"],
                             "validation": validation()},
            "per_step_s": [round(x, 3) for x in vals],
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------
# the product

def roofline_of(kern, nL, peak, config):
    """dominant-kernel roofline from a profiled (per-launch CUDA-event) pass"""
    ksum = kern["gemm_ms"] + kern["carry_ms"] + kern["gather_ms"] + kern["epilogue_ms"] + kern["other_ms"]
    # small systems (order <= 256) run the whole Dixon solve of a pole drop in
    # one launch, larger ones as one dataflow launch per sweep chunk: both
    # products of every digit are in gemm_ms
    fused = kern["carry_launches"] == 0 and kern.get("carry_macs", 0) > 0
    gemm_macs = kern["gemm_macs"] + (kern["carry_macs"] if fused else 0)
    achieved = 2 * gemm_macs / max(1e-9, kern["gemm_ms"] / 1e3) / 1e12
    if not fused:
        kname = "tc::gemm_kernel (digit product y_k = bal(Cq . in_k))"
    elif nL <= 256:
        kname = "tc::dixon_fused_kernel (digit + carry products of every digit, one launch per pole drop)"
    else:
        kname = "tc::dixon_flow_kernel (dense digit + block-sparse carry tiles of every digit, one dataflow launch)"
    traffic = committed_traffic(config)
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)",
            "frac": achieved / peak if peak else None, "traffic": (traffic or {}).get("bytes_per_launch"),
            "traffic_source": (traffic or {}).get("source"), "kernel": kname,
            "avg_launch_ms": kern["gemm_ms"] / max(1, kern["gemm_launches"]),
            "share_of_kernel_time": kern["gemm_ms"] / ksum if ksum else None,
            "peak_source": "measured on this box: torch._int_mm 8192^3 int8 (cuBLASLt), best of 5",
            "macs_per_launch": gemm_macs / max(1, kern["gemm_launches"]),
            "epilogue": {"kernel": "dev::epilogue_kernel (w' = T_x y, carry-normalised digits)",
                         "ms": kern["epilogue_ms"], "share_of_kernel_time": kern["epilogue_ms"] / ksum if ksum else None}}


def matvec_stepping(drzg, torch):
    """north_star (a): achieved HBM GB/s of the reference-shaped linrec_eval
    (linalg.hpp:337-410) on the device, drzg_linrec_eval_device with the inputs
    resident, CUDA events around tmax + 1 = 21 factors, best of 3; algorithmic
    bytes = A and B once per factor (2 side^2 8 limbs); at side 3003 the
    matrices (144 / 289 MB) exceed the 126 MB L2"""
    hbm = measured_peaks().get("hbm_gbs")
    out = []
    for p, M, side in [(7, 20, 3003), (7, 24, 3003), (13, 13, 495)]:
        sp = drzg.stripe_plan(p, M)
        L = sp.limbs
        g = torch.Generator(device="cuda").manual_seed(1)
        hi = min(int(sp.beta), 2**62)
        A = torch.randint(0, hi, (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
        B = torch.randint(0, hi, (L * side * side,), dtype=torch.int64, device="cuda", generator=g)
        w = torch.randint(0, hi, (L * side,), dtype=torch.int64, device="cuda", generator=g)
        if L > 1:
            top = p ** (M - sp.limb_exp * (L - 1))
            for X in (A, B, w):
                X.view(L, -1)[L - 1] %= top
        drzg.linrec_eval_device(p, M, side, A.data_ptr(), B.data_ptr(), 2, w.data_ptr())
        torch.cuda.synchronize()
        best = min(drzg.linrec_eval_device(p, M, side, A.data_ptr(), B.data_ptr(), 20, w.data_ptr(), timed=True)
                   for _ in range(3))
        per = best / 21
        gbs = 2 * side * side * 8 * L / (per / 1e3) / 1e9
        out.append({"p": p, "M": M, "side": side, "limbs": L, "us_per_factor": round(per * 1e3, 2),
                    "alg_GBps": round(gbs, 1), "frac_hbm": round(gbs / hbm, 3) if hbm else None,
                    "kernel": "linrec_flat_kernel" if side * side >= (1 << 20) else "linrec_resident_kernel"})
        del A, B, w
    torch.cuda.empty_cache()
    return {"cases": out, "peak_GBps": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}


def fourfold_leg(drzg, torch, local, peak):
    """ONE complete zeta function of the metric's own hypersurface (configs[4])
    under clock sampling, after a one-column warm-up; then column 0 once more
    with per-launch kernel timing for the roofline"""
    p, n, d, seed, desc = CONFIGS["fourfold"]
    coeffs = drzg.random_hypersurface(p, n, d, seed=seed)
    t0 = time.time()
    drzg.frobenius(p, n, d, coeffs, columns=[0], device=local)  # tables, state pool, allocations
    warm = time.time() - t0
    with ClockSampler(local, "_fourfold") as clk:
        torch.cuda.synchronize()
        clk.mark()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        z = drzg.zeta(p, n, d, coeffs, device=local, count_budget=FOURFOLD_COUNT_BUDGET)
        e1.record()
        torch.cuda.synchronize()
        e2e = e0.elapsed_time(e1) / 1e3
    clocks = clk.summary()
    fr = z["frobenius"]
    ref = full_ledger("fourfold")
    led = {k: fr[k] for k in ("matvecs", "startups", "combines")}
    # the first column group as the pipeline forms it (columns 0-1), per-launch timed
    colp = drzg.frobenius(p, n, d, coeffs, columns=[0, 1], device=local, profile=True)
    kern = colp["kernels"]
    rl = roofline_of(kern, colp["nL"], peak, "fourfold")
    dev_s = fr["kernels"]["device_ms"] / 1e3
    macs = fr["kernels"]["gemm_macs"] + fr["kernels"]["carry_macs"]
    return {
        "workload": desc, "value": z["seconds"], "unit": "s", "e2e": e2e, "warmup_one_column_s": warm,
        "device_s": dev_s, "stage_seconds": fr["times"],
        "engine_int8_tops": 2 * macs / max(1e-9, dev_s) / 1e12,
        "engine_frac_of_int8_peak": (2 * macs / max(1e-9, dev_s) / 1e12) / peak if peak else None,
        "ledger": led, "reference_ledger": ref, "ledger_equal": bool(ref) and all(led[k] == ref[k] for k in led),
        "Q_sha256": hashlib.sha256(json.dumps(z["Q"]).encode()).hexdigest(), "Q_head": z["Q"][:4],
        "counts": z["counts"], "counts_ok": all(ok for (_, _, ok) in z["counts"]) and len(z["counts"]) == 2,
        "slopes": z["slopes"], "escalations": z["escalations"], "clocks": clocks,
        "digits": fr["digits"], "peak_live_states": fr["kernels"]["peak_live_states"],
        "roofline_columns01": rl, "kernels_ms_columns01": kern,
        "gpu_launches": fr["traffic"]["launches"],
        "h2d_bytes": fr["traffic"]["h2d_bytes"], "d2h_bytes": fr["traffic"]["d2h_bytes"],
    }


def fourfold_leg_dist(drzg, torch, dist, world, rank, local):
    """ONE complete zeta function of configs[4] with its columns partitioned
    over the ranks (longest-processing-time on the reference's replayed
    per-column matvecs), F assembled by drzg_gather_F (one ncclAllGather), and
    run_zeta's battery (drzg_zeta_from_F: Q, Newton >= Hodge, both point
    counts) on rank 0.  Time = max over ranks of the whole call sequence.
    Returns the result on rank 0, None elsewhere."""
    from paper_2602_24155_b200 import parallel
    p, n, d, seed, desc = CONFIGS["fourfold"]
    coeffs = drzg.random_hypersurface(p, n, d, seed=seed)
    b = sum(hodge_counts(n, d))
    weights = parallel.replayed_column_weights(os.path.join(GOLD, "ledger_replay_fourfold.json"))
    mine = parallel.partition_columns(n, d, world, rank, weights=weights)
    t0 = time.time()
    drzg.frobenius(p, n, d, coeffs, columns=mine[:1], device=local)  # tables, state pool, allocations
    parallel.nccl_comm(world, rank, local)  # communicator set up outside the timed region
    warm = time.time() - t0
    with ClockSampler(local, "_fourfold") as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        t1 = time.time()
        fr = drzg.frobenius(p, n, d, coeffs, columns=mine, device=local)
        F = parallel.gather_frobenius_nccl(fr["F"], b, mine, world, rank, local)
        z = None
        if rank == 0:
            z = drzg.zeta_from_F(p, n, d, coeffs, [str(x) for x in F], b, count_budget=FOURFOLD_COUNT_BUDGET)
        torch.cuda.synchronize()
        wall = time.time() - t1
    clocks = clk.summary()
    led = [fr["matvecs"], fr["startups"], fr["combines"], fr["kernels"]["device_ms"] / 1e3, wall]
    if dist:
        t = torch.tensor(led[:3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        m = torch.tensor(led[3:], dtype=torch.float64, device="cuda")
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        led = t.tolist() + m.tolist()
    if rank != 0:
        return None
    ref = full_ledger("fourfold")
    mine_led = {"matvecs": int(led[0]), "startups": int(led[1]), "combines": int(led[2])}
    return {
        "workload": desc + f", columns partitioned over {world} GPU(s), F gathered by one ncclAllGather",
        "value": led[4], "unit": "s", "n_gpus": world, "warmup_s": warm, "device_s_max_rank": led[3],
        "status": z["status"], "ledger": mine_led, "reference_ledger": ref,
        "ledger_equal": bool(ref) and all(mine_led[k] == ref[k] for k in mine_led),
        "Q_sha256": hashlib.sha256(json.dumps(z.get("Q")).encode()).hexdigest() if z.get("Q") else None,
        "counts": z.get("counts"), "counts_ok": bool(z.get("counts")) and all(ok for (_, _, ok) in z["counts"]),
        "clocks_rank0": clocks,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="k3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fourfold-leg", default="auto", choices=["auto", "on", "off", "dist"])
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
    budget = FOURFOLD_COUNT_BUDGET if args.config == "fourfold" else 0
    # columns partitioned across ranks (longest-processing-time by pole order)
    from paper_2602_24155_b200 import parallel
    weights = None
    if args.config == "fourfold":  # the reference's replayed per-column work
        weights = parallel.replayed_column_weights(os.path.join(GOLD, "ledger_replay_fourfold.json"))
    all_cols = [parallel.partition_columns(n, d, world, r, weights=weights) for r in range(world)]
    mine = all_cols[rank] if world > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    batch = args.config == "threefold_batch"
    if batch:
        batch_coeffs = [drzg.random_hypersurface(p, n, d, seed=s) for s in range(rank, BATCH_SEEDS, world)]

    def step(profile=False):
        """one zeta function (or the rank's share of a batch); returns
        (zeta-call seconds, result json of this rank, frobenius json)"""
        if batch:
            # BATCH_WORKERS hypersurfaces in flight on their own host threads
            # and streams (zeta_batch); the step's value is its wall time
            t0 = time.time()
            zs = drzg.zeta_batch(p, n, d, batch_coeffs, workers=1 if profile else BATCH_WORKERS, device=local,
                                 profile=profile, verify_counts=True)
            wall = time.time() - t0
            if not all(ok for z_ in zs for (_, _, ok) in z_["counts"]):
                raise RuntimeError("a point count disagrees with Q")
            fr_ = merge_frobenius([z_["frobenius"] for z_ in zs])
            z0 = dict(zs[0], seconds=wall)
            return wall, z0, fr_
        if world == 1:
            z = drzg.zeta(p, n, d, coeffs, r_uniform=r_uniform, device=local, profile=profile,
                          verify_counts=True, count_budget=budget)
            return z["seconds"], z, z["frobenius"]
        t0 = time.time()
        fr = drzg.frobenius(p, n, d, coeffs, r_uniform=r_uniform, columns=mine, device=local, profile=profile)
        # one ncclAllGather of the column blocks issued by libdrzg.so (drzg_gather_F)
        F = parallel.gather_frobenius_nccl(fr["F"], b, mine, world, rank, local)
        z = None
        if rank == 0:
            # run_zeta's battery on the gathered F: Q recovery, sign tie-break,
            # Newton >= Hodge, point counts (the step fails unless it passes)
            z = drzg.zeta_from_F(p, n, d, coeffs, [str(x) for x in F], b, r_uniform=r_uniform,
                                 count_budget=budget)
            if z["status"] != "ok":
                raise RuntimeError(f"gathered F needs escalation: {z['reason']}")
            if not all(ok for (_, _, ok) in z["counts"]):
                raise RuntimeError("a point count disagrees with Q")
        return time.time() - t0, z, fr

    vals, dev_times, e2e_times, last = [], [], [], None
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
            call_s, z, fr = step()
            e1.record()
            torch.cuda.synchronize()
            e2e_s = e0.elapsed_time(e1) / 1e3
            dev_s = fr["kernels"]["device_ms"] / 1e3
            if dist:
                tt = torch.tensor([call_s, e2e_s, dev_s], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                call_s, e2e_s, dev_s = tt.tolist()
            vals.append(call_s)
            e2e_times.append(e2e_s)
            dev_times.append(dev_s)
            last = (z, fr)
    if dist:
        dist.barrier()
    clocks = clk.summary()
    # profiled pass: per-kernel CUDA-event times on the engine stream
    _, _, frp = step(profile=True)
    # the metric's own configuration across all ranks (every rank takes part)
    dist_leg = None
    if args.config == "k3" and (args.fourfold_leg == "dist" or (args.fourfold_leg in ("auto", "on") and world > 1)):
        try:
            dist_leg = fourfold_leg_dist(drzg, torch, dist, world, rank, local)
        except Exception as e:
            dist_leg = {"error": str(e)} if rank == 0 else None
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    z, fr = last
    value = sum(vals) / len(vals)
    e2e = sum(e2e_times) / len(e2e_times)
    kern = frp["kernels"]
    peak = int8_peak_tops(torch)
    rl = roofline_of(kern, fr["nL"], peak, args.config)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refapi
            info = reference_measure(args.config, [int(x) for x in refapi.hypersurface(p, n, d, seed=seed)],
                                     host_threads())
            if info:
                cpu = {"value": info["value"], "unit": "s", "cores": host_threads(), "kind": info["kind"],
                       "projection": info["projection"], "sample": info["sample"], "validation": validation()}
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": "s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    # mod-p^N reduction Gop/s = 2 side^2 per matvec x matvecs / s (engine time)
    dev_mean = sum(dev_times) / len(dev_times)
    gops = 2.0 * fr["side"] ** 2 * fr["matvecs"] / dev_mean / 1e9 if world == 1 else None
    ref_led = full_ledger(args.config)
    srt = sorted(vals)
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
        "engine_device_s": dev_mean,
        "roofline": rl,
        "reduction_gops": gops,
        "ledger": {"matvecs": fr["matvecs"], "startups": fr["startups"], "combines": fr["combines"],
                   "terms": fr["terms"], "reference": ref_led,
                   "equal": bool(ref_led) and all(fr[k] == ref_led[k] for k in ("matvecs", "startups", "combines"))},
        "per_step_s": {"zeta_call": [round(x, 4) for x in vals], "e2e": [round(x, 4) for x in e2e_times],
                       "engine_device": [round(x, 4) for x in dev_times],
                       "median": srt[len(srt) // 2], "p95": srt[min(len(srt) - 1, int(0.95 * len(srt)))]},
        "stage_seconds": fr["times"], "kernels_ms": kern,
        "cpu_baseline": cpu, "clocks": clocks,
        "Q_head": (z["Q"][:4] if z and "Q" in z else None),
    }
    if dist_leg is not None:
        line["fourfold"] = dist_leg
    try:
        line["matvec_stepping"] = matvec_stepping(drzg, torch)
    except Exception as e:
        line["matvec_stepping"] = {"error": str(e)}
    leg = dist_leg is None and (args.fourfold_leg == "on" or (args.fourfold_leg == "auto" and world == 1 and
                                                               args.config == "k3"))
    if leg:
        try:
            line["fourfold"] = fourfold_leg(drzg, torch, local, peak)
            ff_cpu = None
            if not args.no_cpu_baseline:
                from oracle import refapi
                info = reference_measure("fourfold", [int(x) for x in refapi.hypersurface(7, 5, 3, seed=1)],
                                         host_threads())
                if info:
                    ff_cpu = {"value": info["value"], "unit": "s", "cores": host_threads(), "kind": info["kind"],
                              "projection": info["projection"], "sample": info["sample"]}
            line["fourfold"]["cpu_baseline"] = ff_cpu
        except Exception as e:
            line["fourfold"] = {"error": str(e)}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
