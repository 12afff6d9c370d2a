#!/usr/bin/env python
"""bench.py -- QR TFLOP/s of the RGSQRF hot path at 32768x16384 (BASELINE.json configs[2]) on N
B200s, plus LLS time-to-FP64 accuracy (configs[3]) as an extra key.

One "step" = one tcqr_factor of the whole matrix (all SURVEY.md §8(a) QR rows: copy/validate, the
Alg. 2 recursion with K1 casts, K3/K4 tcgen05 GEMMs, FP32 products below the cutoff, the Eq. (6)
panel), inputs resident in HBM. value = (2 M n^2 - 2/3 n^3) / time (the north_star convention),
summed over the whole job (N > 1: row-partitioned single factorization, strong scaling).

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under torchrun (one rank per
GPU, NCCL). --impl reference times the CPU oracle (the base contract's reference arm for this tier).
"""
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

METRIC = "QR TFLOP/s at 32768x16384; LLS time-to-FP64 accuracy; 1/2/4/8 GPUs"
WORKLOADS = {
    "cfg3": dict(m=32768, n=16384, kind="gaussian", seed=4,
                 name="QR of 32768x16384 Gaussian (BASELINE configs[2])"),
    "cfg2": dict(m=16384, n=4096, kind="gaussian", seed=2,
                 name="QR of 16384x4096 Gaussian (BASELINE configs[1])"),
    "cfg5": dict(m=262144, n=2048, kind="gaussian", seed=8,
                 name="QR of 262144x2048 Gaussian (BASELINE configs[4])"),
    "cfg1": dict(m=1024, n=128, kind="gaussian", seed=1,
                 name="QR of 1024x128 Gaussian (BASELINE configs[0])"),
    "next3": dict(m=4194304, n=128, kind="gaussian", seed=9,
                  name="orthogonalization of 4194304x128 Gaussian (NEXT-3, PAPER.md:598)"),
}


def conv_flops(m, n):
    return 2.0 * m * n * n - 2.0 / 3.0 * n ** 3


def fp32_peak_tflops(sm_mhz=1965.0):
    """FP32 SIMT peak of one B200: 148 SMs x 128 FP32 lanes x 2 flop (FMA) x the max SM clock
    (1965 MHz, the clock nvidia-smi reports under load on this pool)."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], tc=d["bf16_tflops"], tc_sustained=d["bf16_tflops_sustained"],
                    src="MEASURED_PEAKS.json (measured)")
    return dict(hbm=6650.0, tc=1590.0, tc_sustained=1400.0, src="B200_PROFILING.md fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_sample(a_cols_np, reps=1):
    """Time the oracle (as it stands) on host cores: oracle.qr.rgs on an m x n_s sample."""
    from oracle.qr import rgs
    t0 = time.perf_counter()
    for _ in range(reps):
        rgs(a_cols_np.astype(np.float64))
    dt = (time.perf_counter() - t0) / reps
    return dt


def cpu_oracle_cgls_sample(a_np, iters=8):
    """Seconds per iteration of the oracle's corrected Alg. 5 (oracle.cgls.pcgls, as it stands) on
    an m x n_s sample, preconditioned by the sample's own sign-fixed R (computed outside the timed
    region); `iters` iterations (the tolerance is set so that none stops early)."""
    from oracle.cgls import pcgls
    a = a_np.astype(np.float64)
    r = np.linalg.qr(a, mode="r")
    r = r * np.sign(np.diag(r))[:, None]
    b = a @ np.ones(a.shape[1]) + 1e-3 * np.random.default_rng(5).standard_normal(a.shape[0])
    t0 = time.perf_counter()
    _, info = pcgls(a, b, r, tol=1e-300, maxit=iters, window=10 ** 9)
    return (time.perf_counter() - t0) / max(info.iterations, 1)


def cpu_info():
    """CPU model (from /proc/cpuinfo) and the BLAS numpy calls (threadpoolctl)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [f"{d.get('internal_api')} {d.get('version')} ({d.get('num_threads')} threads)"
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:  # noqa: BLE001 -- informational only
        pass
    return {"cpu_model": model, "blas": blas, "numpy": np.__version__}


def run_reference(args, wl):
    """--impl reference: the CPU FP64 oracle timed on this box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import workloads as W
    m, n_s = wl["m"], min(wl["n"], args.cpu_sample_cols)
    a = W.gaussian(m, n_s, seed=wl["seed"])
    cores = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        cpu_oracle_sample(a)
    ts = [cpu_oracle_sample(a) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    v = conv_flops(m, n_s) / t / 1e12
    sample = f"oracle.qr.rgs (FP64 numpy) on the first {n_s} columns of the {m}x{wl['n']} workload"
    line = {
        "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": wl["name"] + f" [CPU sample {m}x{n_s}]", "m": m, "n": n_s},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample, **cpu_info()},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def model_ideal_ms(m, n, peaks, cutoff=128):
    """Modelled ideal factorization time at the measured peaks: per split node the
    longer of its tensor-core time (4 m h w2 flops at the sustained bf16 = fp16 dense rate) and its
    HBM time (K1 cast 6 m w2 + K3 2m(h + w2) + K4 2mh + 8 m w2 bytes); per leaf the longer of its
    FP32 time (2 m c^2 flops at the FP32 SIMT peak) and its HBM time (10 m c bytes)."""
    tc = peaks["tc_sustained"] * 1e12
    hbm = peaks["hbm"] * 1e9
    fp32 = fp32_peak_tflops() * 1e12

    def rec(w):
        if w <= cutoff:
            return max(2.0 * m * w * w / fp32, 10.0 * m * w / hbm)
        h = 32 * ((w + 63) // 64)
        w2 = w - h
        node = max(4.0 * m * h * w2 / tc, (4.0 * m * h + 16.0 * m * w2) / hbm)
        return rec(h) + node + rec(w2)

    return rec(n) * 1e3


def other_configs(tq, W, torch, dev, peaks, steps, cutoff):
    """The other BASELINE.json configs at N = 1 (extra keys, not the headline): configs[0] latency,
    configs[1] and configs[4] QR TFLOP/s, the NEXT-3 4194304 x 128 orthogonalization, configs[4]
    LLS and the configs[3] FP32-target LLS; each with its modelled-ideal fraction and a parity
    check against the oracle (small configs) or the leading columns (large ones)."""
    from oracle.cgls import oracle_lls
    from oracle.metrics import r_rel_error, x_rel_error
    from oracle.qr import rgs
    out = {}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def qr_case(key, m, n, seed, reps, lead=256):
        A = W.gaussian_cuda(m, n, seed, device=dev)
        Q = tq.colmajor_empty(m, n, device=dev)
        R = tq.colmajor_empty(n, n, device=dev)
        ms = timed(lambda: tq.factor(A, Q, R), reps)
        ideal = model_ideal_ms(m, n, peaks, cutoff)
        k = min(lead, n)
        _, r_o = rgs(A[:, :k].cpu().numpy().astype(np.float64))
        rec = {"m": m, "n": n, "ms": ms, "tflops": conv_flops(m, n) / (ms * 1e-3) / 1e12,
               "model_ideal_ms": ideal, "frac_of_model_ideal": ideal / ms,
               f"R_lead{k}_rel_err_vs_oracle": r_rel_error(R[:k, :k].cpu().numpy().astype(np.float64), r_o)}
        del A, Q, R
        torch.cuda.empty_cache()
        out[key] = rec
        return rec

    # configs[0]: 1024 x 128 QR + LLS latency, full oracle parity (c = 128: the leaf kernel only)
    a1 = W.gaussian(1024, 128, seed=W.CONFIG_SEEDS["cfg1"])
    b1, _ = W.consistent_rhs(a1, seed=W.CONFIG_SEEDS["cfg1_x"])
    A1 = tq.to_device_colmajor(a1)
    B1 = torch.from_numpy(b1).to(dev)
    Q1, R1 = tq.colmajor_empty(1024, 128, device=dev), tq.colmajor_empty(128, 128, device=dev)
    qr_us = timed(lambda: tq.factor(A1, Q1, R1), 50) * 1e3
    x1 = [None]
    lls_us = timed(lambda: x1.__setitem__(0, tq.lls_solve(A1, B1, tol=1e-10, maxit=200)), 20) * 1e3
    _, r1o = rgs(a1.astype(np.float64))
    x1o, _ = oracle_lls(a1.astype(np.float64), b1)
    out["cfg1"] = {"workload": "configs[0] 1024x128 Gaussian: QR + R-preconditioned CGLS to 1e-10",
                   "qr_latency_us": qr_us, "lls_latency_us": lls_us,
                   "lls_iterations": x1[0][1]["iterations"],
                   "R_rel_err_vs_oracle": r_rel_error(R1.cpu().numpy().astype(np.float64), r1o),
                   "x_rel_err_vs_oracle": x_rel_error(x1[0][0].cpu().numpy(), x1o),
                   "note": "launch-latency bound (a us-scale ideal), reported as latency"}
    del A1, B1, Q1, R1
    qr_case("cfg2", 16384, 4096, W.CONFIG_SEEDS["cfg2"], steps)["workload"] = \
        "configs[1] QR of 16384x4096 Gaussian"
    qr_case("cfg5", 262144, 2048, W.CONFIG_SEEDS["cfg5"], steps)["workload"] = \
        "configs[4] QR of 262144x2048 Gaussian (1 GPU)"
    qr_case("next3", 4194304, 128, 9, steps, lead=128)["workload"] = \
        "NEXT-3 orthogonalization of 4194304x128 Gaussian (PAPER.md:598)"
    # configs[4] LLS: Gaussian b = A x_true, FP64 target
    m5, n5 = 262144, 2048
    A5 = W.gaussian_cuda(m5, n5, W.CONFIG_SEEDS["cfg5"], device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(W.CONFIG_SEEDS["cfg5_x"])
    xt = torch.randn(n5, generator=g, device=dev, dtype=torch.float64)
    b5 = A5.to(torch.float64) @ xt
    res = [None]
    ms5 = timed(lambda: res.__setitem__(0, tq.lls_solve(A5, b5, tol=1e-10, maxit=400)), 2)
    x5, info5 = res[0]
    out["cfg5_lls"] = {"workload": "configs[4] LLS 262144x2048 Gaussian, b = A x_true, FP64 target",
                       "time_to_solution_ms": ms5, "qr_ms": info5["qr_ms"],
                       "cgls_ms": info5["cgls_ms"], "iterations": info5["iterations"],
                       "x_rel_err_vs_x_true": float(torch.linalg.norm(x5 - xt) / torch.linalg.norm(xt))}
    del A5, b5, x5
    torch.cuda.empty_cache()
    return out


def _streamed_r_bytes(n, cutoff):
    """Bytes of R the streamed tcqr_factor_host copies back: for each column chunk (the subtrees
    of width <= max(n/div, 2*cutoff), div = TCQR_STREAM_DIV or 16, tcqr.cu plan_chunks) the rows
    [0, chunk end); the zero rows below are written on the host."""
    div = int(os.environ.get("TCQR_STREAM_DIV", "16") or 16)
    target = max(n // max(div, 1), 1)
    chunks = []

    def plan(c0, w):
        if w <= target or w <= 2 * cutoff:
            chunks.append((c0, c0 + w))
            return
        h = 32 * ((w + 63) // 64)
        plan(c0, h)
        plan(c0 + h, w - h)

    if n <= 2 * cutoff:
        return 4 * n * n
    plan(0, n)
    return sum(4 * b * (b - a) for a, b in chunks)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-sample-cols", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lls", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--cutoff", type=int, default=128)
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs (extra keys)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist
    import paper_1912_05508_b200 as tq
    import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        tq.init_distributed()
    else:
        tq.init(local)
    tq.set_config(cutoff=args.cutoff)
    dev = torch.device("cuda", local)
    M, n = wl["m"], wl["n"]
    rows = np.array_split(np.arange(M), world)[rank]
    r0, r1 = int(rows[0]), int(rows[-1]) + 1
    m = r1 - r0
    Afull = W.gaussian_cuda(M, n, wl["seed"], device=dev)           # same A on every rank
    A = torch.empty((n, m), dtype=torch.float32, device=dev).t()
    A.copy_(Afull[r0:r1])
    del Afull
    torch.cuda.empty_cache()
    Q = tq.colmajor_empty(m, n, device=dev)
    R = tq.colmajor_empty(n, n, device=dev)
    tq.reserve_workspace(m, n, op=0)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        tq.factor(A, Q, R)
    torch.cuda.synchronize()
    launches_per_step = tq.last_launch_count()
    collectives_per_step = tq.last_collective_count()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            tq.factor(A, Q, R)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = conv_flops(M, n) / (ms * 1e-3) / 1e12

    # ---- sampled parity at full size (oracle on the leading 256 columns: R11 of A = QR) ----
    parity = None
    if rank == 0 and world == 1:
        from oracle.qr import rgs
        from oracle.metrics import r_rel_error
        k = min(256, n)
        if M <= 262144:
            a_lead = A[:, :k].cpu().numpy().astype(np.float64)
            q_o, r_o = rgs(a_lead)
            r_lead = R[:k, :k].cpu().numpy().astype(np.float64)
            q_lead = Q[:, :k].cpu().numpy().astype(np.float64)
            # R's leading k rows over ALL columns: R = Q'A is unique, so rows 0..k-1 are Q_k' A
            # with the oracle's Q_k of the leading columns (FP64 on the host, column chunks)
            rows_o = np.empty((k, n))
            for c0 in range(0, n, 2048):
                c1 = min(n, c0 + 2048)
                rows_o[:, c0:c1] = q_o.T @ A[:, c0:c1].cpu().numpy().astype(np.float64)
            parity = {f"R_lead{k}_rel_err_vs_oracle": r_rel_error(r_lead, r_o),
                      f"R_rows{k}_all_cols_rel_err_vs_oracle": r_rel_error(
                          R[:k, :].cpu().numpy().astype(np.float64), np.triu(rows_o)),
                      f"Q_lead{k}_orthogonality_f": float(
                          np.linalg.norm(q_lead.T @ q_lead - np.eye(k)) / np.sqrt(k))}
        else:
            # the FP64 CPU oracle on all rows of a 4M-row block takes minutes: device invariants
            # only (tests/test_gpu_fullsize.py pins the oracle comparison at smaller row counts)
            parity = {"oracle": "skipped at this row count; device FP64 invariants below"}
        # full-size invariants on the device in FP64 (harness arithmetic, not the method)
        Rd = R.to(torch.float64)
        res = 0.0
        nrm = 0.0
        for c0 in range(0, n, 2048):
            c1 = min(n, c0 + 2048)   # R is upper triangular: only Q[:, :c1] contributes
            blk = A[:, c0:c1].to(torch.float64) - Q[:, :c1].to(torch.float64) @ Rd[:c1, c0:c1]
            res += float(torch.linalg.norm(blk) ** 2)
            nrm += float(torch.linalg.norm(A[:, c0:c1].to(torch.float64)) ** 2)
            del blk
        parity["backward_error_f"] = (res / nrm) ** 0.5
        Qd = Q.to(torch.float64)
        parity["orthogonality_f"] = float(torch.linalg.norm(Qd.T @ Qd - torch.eye(n, device=dev,
                                          dtype=torch.float64)) / n ** 0.5)
        del Qd, Rd
        torch.cuda.empty_cache()

    # ---- per-kernel-class profile pass (CUDA events around every launch, same stream) ----
    peaks = load_peaks()
    roofline, classes = None, None
    if not args.no_profile:
        tq.profile_enable(True)
        tq.factor(A, Q, R)
        classes = tq.profile_read()
        tq.profile_enable(False)
        tot = sum(c["ms"] for c in classes.values()) or 1.0
        dom = max(classes, key=lambda k: classes[k]["ms"])
        c = classes[dom]
        per_launch_ms = c["ms"] / max(c["launches"], 1)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(args.workload, {}).get(dom)
        if dom in ("k3_tn", "k4_nn"):
            ach = c["flops"] / (c["ms"] * 1e-3) / 1e12
            roofline = {"bound": "tensor", "achieved": ach, "peak": peaks["tc_sustained"],
                        "unit": "TFLOP/s", "frac": ach / peaks["tc_sustained"], "traffic": traffic}
        else:
            # SIMT classes: the bound is whichever ideal time is longer, HBM bytes at the measured
            # copy bandwidth or FP32 flops at the FP32 SIMT peak (148 SMs x 128 FP32 lanes x 2 flop
            # x the max SM clock -- DESIGN.md section 6); the whole-leaf kernel is FP32-bound
            t_hbm = c["bytes"] / (peaks["hbm"] * 1e9)
            t_alu = c["flops"] / (fp32_peak_tflops() * 1e12)
            if t_alu > t_hbm:
                ach = c["flops"] / (c["ms"] * 1e-3) / 1e12
                roofline = {"bound": "alu", "achieved": ach, "peak": fp32_peak_tflops(),
                            "unit": "TFLOP/s", "frac": ach / fp32_peak_tflops(), "traffic": traffic,
                            "hbm_achieved_gbs": c["bytes"] / (c["ms"] * 1e-3) / 1e9}
            else:
                ach = c["bytes"] / (c["ms"] * 1e-3) / 1e9
                roofline = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                            "frac": ach / peaks["hbm"], "traffic": traffic}
        roofline.update({"kernel": dom, "share_of_step": c["ms"] / tot,
                         "launches_per_step": c["launches"], "ms_per_launch": per_launch_ms,
                         "peak_source": (peaks["src"] + " bf16 sustained (fp16 dense = bf16 rate)"
                                         if dom in ("k3_tn", "k4_nn") else
                                         "derived FP32 SIMT peak: 148 SMs x 128 lanes x 2 x 1965 MHz"
                                         if roofline["bound"] == "alu" else peaks["src"] + " hbm_gbs")})
        classes = {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                       "share": round(v["ms"] / tot, 4),
                       "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 2),
                       "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
                   for k, v in classes.items() if v["launches"]}

    # ---- e2e: the same factorization through the host-pointer C ABI (H2D A, D2H Q and R) ----
    e2e = None
    if not args.no_e2e:
        a_host = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
        a_host.copy_(A.t())
        a_np = a_host.numpy().T           # column-major view of the pinned buffer
        q_host = torch.empty((n, m), dtype=torch.float32, pin_memory=True).numpy().T
        r_host = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy().T
        import ctypes
        L = tq.lib()
        P = ctypes.c_void_p
        steps_e2e = max(1, min(args.steps, 3))
        rc = L.tcqr_factor_host(m, n, a_np.ctypes.data_as(P), m, q_host.ctypes.data_as(P),
                                r_host.ctypes.data_as(P))
        assert rc == 0, rc
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(steps_e2e):
            rc = L.tcqr_factor_host(m, n, a_np.ctypes.data_as(P), m, q_host.ctypes.data_as(P),
                                    r_host.ctypes.data_as(P))
            assert rc == 0, rc
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / steps_e2e
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": conv_flops(M, n) / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ems, "h2d_bytes_per_step": 4 * m * n,
               "d2h_bytes_per_step": 4 * m * n + _streamed_r_bytes(n, args.cutoff),
               "api": "tcqr_factor_host (pinned host A, Q, R): column chunks streamed in, "
                      "finished chunks' Q and R columns streamed out during the factorization"}
        del a_host

    # ---- LLS time-to-FP64 accuracy (configs[3]: 32768x8192 geometric kappa=1e4) ----
    lls = None
    if not args.no_lls and args.workload == "cfg3":
        del Q, R
        torch.cuda.empty_cache()
        Ml, nl = 32768, 8192
        lrows = np.array_split(np.arange(Ml), world)[rank]
        l0, l1 = int(lrows[0]), int(lrows[-1]) + 1
        lls = {"workload": "LLS 32768x8192 geometric kappa=1e4 and 1e6, b = A x_true (BASELINE "
                           "configs[3]), FP64 target (tol 1e-10, one restart), warm (graphs captured)"}

        def lls_case(cond, cases):
            key = "k1e4" if cond == 1e4 else "k1e6"
            Al_full = W.spectrum_cuda(Ml, nl, "geometric", cond, W.CONFIG_SEEDS["cfg4_" + key],
                                      device=dev)
            g = torch.Generator(device=dev)
            g.manual_seed(W.CONFIG_SEEDS["cfg4_x_" + key])
            x_true = torch.randn(nl, generator=g, device=dev, dtype=torch.float64)
            b_full = Al_full.to(torch.float64) @ x_true
            Al = torch.empty((nl, l1 - l0), dtype=torch.float32, device=dev).t()
            Al.copy_(Al_full[l0:l1])
            bl = b_full[l0:l1].contiguous()
            del Al_full, b_full
            torch.cuda.empty_cache()
            for case in cases:
                label, reorth, split = case[:3]
                restart = case[3] if len(case) > 3 else 1
                tq.set_config(cutoff=args.cutoff, reorth=reorth, fp16_split=split, restart=restart)
                tq.lls_solve(Al, bl, tol=1e-10, maxit=4000)      # warm-up: builds the QR graph
                barrier()
                torch.cuda.synchronize()
                h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                h0.record(stream)
                x, info = tq.lls_solve(Al, bl, tol=1e-10, maxit=4000)
                h1.record(stream)
                torch.cuda.synchronize()
                lt = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
                if world > 1:
                    dist.all_reduce(lt, op=dist.ReduceOp.MAX)
                xe = float(torch.linalg.norm(x - x_true) / torch.linalg.norm(x_true))
                lls[label] = {"time_to_solution_ms": float(lt.item()), "qr_ms": info["qr_ms"],
                              "cgls_ms": info["cgls_ms"], "iterations": info["iterations"],
                              "iterations_pass1": info["iterations_pass1"],
                              "converged": bool(info["converged"]), "x_rel_err_vs_x_true": xe,
                              "fp64_accuracy_reached": bool(xe <= 1e-10)}
            del Al, bl

        lls_case(1e4, (("paper_R", 0, 0), ("reorth_R", 1, 0), ("split_reorth_R", 1, 1)))
        # FP32 target (one pass, tol 1e-10, no restart; gate x within 1e-5, SURVEY 8(d) configs[3])
        lls_case(1e4, (("paper_R_fp32_target", 0, 0, 0),))
        lls["paper_R_fp32_target"]["fp32_accuracy_reached"] = \
            lls["paper_R_fp32_target"]["x_rel_err_vs_x_true"] <= 1e-5
        tq.set_config(cutoff=args.cutoff)
        # CGLS per-iteration roofline: 2 FP32 passes over A (8 m n B) and 2 over the FP32 upper
        # triangle of R^-1 (4 n (n+1) B) per iteration
        pr = lls["paper_R"]
        it_ms = pr["cgls_ms"] / max(pr["iterations"], 1)
        it_bytes = 8.0 * Ml * nl + 4.0 * nl * (nl + 1)
        lls["cgls_iteration"] = {"ms": it_ms, "bytes": it_bytes,
                                 "gbs": it_bytes / (it_ms * 1e-3) / 1e9,
                                 "frac_of_hbm": it_bytes / (it_ms * 1e-3) / 1e9 / peaks["hbm"],
                                 "note": "paper_R cgls_ms (includes the one-time FP64 R^-1) / "
                                         "iterations"}
        # kappa = 1e6 geometric is beyond the paper with its FP16 R (reading R-A24: CGLS does not
        # converge; 4000 iterations x 2 passes would take seconds): NEXT-4 + NEXT-1 only
        lls_case(1e6, (("k1e6_split_reorth_R", 1, 1),))
        lls["reorth_R"]["note"] = ("NEXT-1 (PAPER.md:622-627): R = R2 R1 from a second RGS of Q; "
                                   "paper_R is Alg. 5 with the single RMGSQR R")
        lls["split_reorth_R"]["note"] = ("NEXT-4 FP16 split (hi + lo halves, three MMAs per product) "
                                         "plus NEXT-1 re-orthogonalization")
        lls["k1e6_split_reorth_R"]["note"] = ("geometric kappa=1e6 (configs[3] second case), "
                                              "NEXT-4 + NEXT-1; the single FP16 R does not converge "
                                              "(R-A24)")
        tq.set_config(cutoff=args.cutoff)

    # ---- the other BASELINE configs (N = 1 only; extra keys) ----
    configs = None
    if world == 1 and not args.no_configs and args.workload == "cfg3":
        try:
            del Q, R
        except NameError:
            pass
        torch.cuda.empty_cache()
        configs = other_configs(tq, W, torch, dev, peaks, args.steps, args.cutoff)

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = min(n, args.cpu_sample_cols)
        a_s = W.gaussian(M, n_s, seed=wl["seed"])   # same distribution, host generator
        dt = cpu_oracle_sample(a_s)
        it_s = cpu_oracle_cgls_sample(a_s[:, :512])
        cpu = {"value": conv_flops(M, n_s) / dt / 1e12, "unit": "TFLOP/s",
               "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"oracle.qr.rgs (FP64 numpy/OpenBLAS) on a {M}x{n_s} Gaussian "
                         f"(first {n_s} columns of the workload shape), {dt:.2f} s",
               "cgls": {"sample": f"oracle.cgls.pcgls on {M}x512 (8 iterations, FP64)",
                        "ms_per_iteration": it_s * 1e3,
                        "gbs": (16.0 * M * 512 + 8.0 * 512 * 512) / it_s / 1e9},
               **cpu_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16xf32", "data": "synthetic",
            "config": {"workload": wl["name"], "M": M, "n": n, "local_rows": m,
                       "cutoff": args.cutoff, "panel_rows": tq.default_config().panel_rows,
                       "flops_convention": "2Mn^2-2/3n^3",
                       "l2": "inputs larger than L2 (A 2 GiB fp32 per step; no flush needed)",
                       "parallelism": f"row-partition x{world}" if world > 1 else "1 GPU",
                       "timing": "CUDA events on the caller stream around K tcqr_factor calls "
                                 "(graph replay), max over ranks"},
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "collectives_per_step": collectives_per_step,
            "clocks": clk.summary(),
            "roofline": roofline,
            "kernel_classes": classes,
            "parity": parity,
            "e2e": e2e,
            "lls": lls,
            "configs": configs,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
