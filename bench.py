"""Benchmark of the FD-apply hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3|4]

One "step" = one fd_apply z = P^{-1} r (Algorithm 1 steps 2-4, PAPER.md 955-964)
over the whole synthetic workload.  Default workload: BASELINE config 4 (d=3,
p=6, n_el=128 per direction: 132^3 x 133 = 305,895,744 DOFs, 2.45 GB per vector)
-- the configuration the metric's "1/2/4/8 B200" is quoted on; it fits one GPU.
For N > 1 the same global problem is slab-partitioned along time over the ranks
("scaling": "strong"), the time mode running after an NCCL all-to-all.

Printed (rank 0): ONE JSON line with value = whole-job DOF/s, the roofline of the
dominant kernel (fd_mode_kernel, FP64 DMMA; peak = the best measured register-only
DMMA rate, profiles/peaks_fp64_r01.json), e2e through fd_apply_host, the oracle
CPU baseline, secondary PCG solve times, clocks.

`--gpus N` without a torchrun environment re-launches itself as N ranks under
torch.distributed.run; `--dry-run` exercises that distributed harness on CPU (gloo).
"""

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

import synth  # noqa: E402

def _fp64_peak():
    """The FP64 roofline denominator: the best measured register-only DMMA.8x8x4 rate
    (tools/fp64_peak.cu on this pool's B200, profiles/peaks_fp64_r01.json; MEASURED_PEAKS.json
    has no FP64 entry).  Fallback: 37.0 TF/s, the same measurement rounded."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")) as f:
            micro = json.load(f)["micro"]
        v = max(m["tflops"] for m in micro if m["kernel"].startswith("dmma"))
        return float(v), ("measured: tools/fp64_peak.cu DMMA.8x8x4 register-only, 148 SMs, best of "
                          "profiles/peaks_fp64_r01.json")
    except Exception:
        return 37.0, "fallback 37.0 (profiles/peaks_fp64_r01.json unreadable)"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = _fp64_peak()


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(cfg_id):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per fd_mode_kernel launch, from the
    committed --set full capture summary (tools/traffic_from_ncu.py -> profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[f"config{cfg_id}"]
        return t["bytes_per_launch"], t["source"]
    except Exception:
        return None, None


def _config_dict(cfg_id, world, a2a="nccl"):
    """The `config` object of the JSON line (identical for both arms)."""
    w = workload(cfg_id)
    return {"workload": f"config{cfg_id}", "d": w["d"], "p": w["p"], "n_el": w["n_el"],
            "n_s": w["n_s"], "n_t": w["n_t"], "N": w["N"],
            "l2": f"inputs larger than L2 ({w['N'] * 8 / 1e9:.2f} GB per vector vs 126 MB)",
            "parallelism": f"time-slab x{world}" if world > 1 else "single GPU",
            "all_to_all": a2a if world > 1 else None}


def fd_flops(d, n_s, n_t, N, cs=True):
    """Algorithmic flops of one fd_apply as executed: 2 n^2 per column of every mode product
    (PAPER.md 1071-1072: 4N(d n_s + n_t) in all); with the centrosymmetric split of the spatial
    modes (ls_tune LS_TUNE_FD_CS, default) a spatial product is two half-size products,
    2 (he^2 + ho^2) per column, he = ceil(n/2), ho = floor(n/2)."""
    he, ho = (n_s + 1) // 2, n_s // 2
    per_space = 2.0 * (he * he + ho * ho) / n_s if cs else 2.0 * n_s
    return 2.0 * N * (d * per_space + 2.0 * n_t)


def workload(cfg_id):
    c = synth.CONFIGS[cfg_id]
    d, p, n_el = c["d"], c["p"], c["n_el"]
    n_s, n_t = n_el + p - 2, n_el + p - 1
    N = n_s ** d * n_t
    flops_paper = 4.0 * N * (d * n_s + n_t)  # PAPER.md 1071-1072
    return {"d": d, "p": p, "n_el": n_el, "n_s": n_s, "n_t": n_t, "N": N, "flops_paper": flops_paper,
            "flops": fd_flops(d, n_s, n_t, N)}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:  # NVML: ~1 ms per sample, so even a sub-second timed region gets many samples
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.rows.append([str(sm), str(mx), str(pw)] +
                                 ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


_SHARE_CACHE = {}


def oracle_share(cfg_id, parts=8, seed=0):
    """One bounded sample of the workload for the CPU oracle: rank 0's share of a `parts`-way
    time-slab split of config `cfg_id`'s fd_apply, computed with the oracle's own functions
    (oracle/fd.py: mode_apply, divisor) as they stand -- the forward spatial modes on time
    slices [0, n_t/parts), the time mode (U_t^T, divide, U_t) on spatial columns [0, N_s/parts),
    the backward spatial modes on the slab.  Every mode runs at its full extent (the per-DOF
    flop count 4(d n_s + n_t) of the full configuration, PAPER.md 1071), on exactly 1/parts
    of the DOFs.  Returns (seconds, DOFs processed, description)."""
    from oracle import univariate as uv, fd
    w = workload(cfg_id)
    d, p, n_el, n_s, n_t = w["d"], w["p"], w["n_el"], w["n_s"], w["n_t"]
    Ns = n_s ** d
    nt_sl, nc = -(-n_t // parts), -(-Ns // parts)
    key = (cfg_id, parts, seed)
    if key not in _SHARE_CACHE:  # setup and inputs once (not part of a step)
        sf, tf = uv.space_factors(n_el, p), uv.time_factors(n_el, p)
        fdd = fd.setup([sf] * d, tf)
        _SHARE_CACHE.clear()
        _SHARE_CACHE[key] = (fdd, synth.residual((nt_sl,) + (n_s,) * d, seed), synth.residual((n_t, nc), seed + 1),
                             np.ascontiguousarray(fd.divisor(fdd).reshape(n_t, Ns)[:, :nc]))
    fdd, r, X, D = _SHARE_CACHE[key]
    t0 = time.perf_counter()
    s = r
    for k in range(1, d + 1):
        s = fd.mode_apply(s, fdd["U_s"][k - 1].T, d + 1 - k)
    q = fd.mode_apply(fd.mode_apply(X, fdd["U_t"].T, 0) / D, fdd["U_t"], 0)
    for k in range(1, d + 1):
        s = fd.mode_apply(s, fdd["U_s"][k - 1], d + 1 - k)
    dt = time.perf_counter() - t0
    assert np.isfinite(s).all() and np.isfinite(q).all()
    dofs = w["N"] / parts
    desc = (f"oracle (numpy tensordot, fp64) on 1/{parts} of config {cfg_id} (N = {w['N']}): the per-rank "
            f"share of a {parts}-way time-slab split -- forward/backward spatial modes on {nt_sl} of {n_t} "
            f"time slices and the time mode on {nc} of {Ns} spatial columns, every mode at full extent "
            f"(same flops per DOF as the full config); DOF/s = (N/{parts}) / time")
    return dt, dofs, desc


def oracle_sample(cfg_id, seconds_min=10.0, max_reps=8):
    """cpu_baseline: oracle_share repeated for >= seconds_min of CPU work; (DOF/s, sample, cores)."""
    oracle_share(cfg_id)  # warm (setup, page faults)
    reps, tot, dofs, desc = 0, 0.0, 0.0, ""
    while reps < max_reps and (reps == 0 or tot < seconds_min):
        dt, n, desc = oracle_share(cfg_id)
        tot += dt
        dofs += n
        reps += 1
    cores = len(os.sched_getaffinity(0))
    return dofs / tot, f"{desc}; {reps} samples, {tot / reps:.2f} s each", cores


def oracle_extras():
    """SURVEY 8(d) "Oracle timing": the oracle fd_apply on one thread (the paper's
    single-thread discipline, PAPER.md 1106) on the same bounded sample as cpu_baseline, and
    oracle PCG solves: config 2 in full (kind 0) and config 5 p = 2 on its spatial grid with
    the time direction truncated to 8 elements (per-iteration time; the full solve would take
    minutes on the host).  A reported baseline, not the target."""
    from threadpoolctl import threadpool_limits
    from oracle import univariate as uv, fd, operator as op, rhs as orhs, pcg as opcg
    out = {}
    with threadpool_limits(limits=1):
        v, sample, _ = oracle_sample(4, seconds_min=5.0, max_reps=2)
    out["oracle_fd_1thread"] = {"value": v, "unit": "DOF/s", "cores": 1, "sample": sample}
    for cfg, p, n_el_t, kind in ((2, 3, 64, 0), (5, 2, 8, 1)):
        d, n_el = synth.CONFIGS[cfg]["d"], synth.CONFIGS[cfg]["n_el"]
        space = [uv.space_factors(n_el, p)] * d
        tf = uv.time_factors(n_el_t, p)
        fdd = fd.setup(space, tf)
        b = orhs.rhs(kind, [space[0]["knots"]] * d, p, tf["knots"], p)
        t0 = time.perf_counter()
        _, it, ok, _ = opcg.pcg(lambda x: op.apply_A(x, space, tf), lambda r: fd.fd_apply(r, fdd), b,
                                max_iter=1000 if cfg == 2 else 3)
        dt = time.perf_counter() - t0
        out[f"oracle_pcg_config{cfg}"] = {
            "N": int(b.size), "iters": it, "solve_s": dt, "s_per_iter": dt / max(it, 1),
            "cores": len(os.sched_getaffinity(0)),
            "sample": ("full config 2, kind 0" if cfg == 2 else
                       f"config 5 p = 2 spatial grid, time truncated to n_el_t = {n_el_t}, first 3 iterations")}
    return out


def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores; each step is one
    oracle_share sample (1/8 of the configuration's DOFs at full per-DOF work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workload(args.config)
    for _ in range(args.warmup):
        oracle_share(args.config)
    tot, dofs, desc = 0.0, 0.0, ""
    for _ in range(args.steps):
        dt, n, desc = oracle_share(args.config)
        tot += dt
        dofs += n
    cores = len(os.sched_getaffinity(0))
    val = dofs / tot
    ms = tot / max(args.steps, 1) * 1e3
    line = {"impl": "reference", "metric": "fd_apply DOF/s (fp64)", "value": val, "unit": "DOF/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(args.config, args.gpus),
            "sample": {"dofs_per_step": dofs / max(args.steps, 1), "of_N": w["N"], "what": desc},
            "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": cores, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _respawn(args):
    """`bench.py --gpus N` (N > 1) without a torchrun environment: re-launch this command as N
    ranks under torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) and pass
    rank 0's JSON line through.  NCCL's environment (NCCL_DEBUG etc.) is inherited unchanged."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.run(cmd).returncode


def run_dry(args):
    """--dry-run: the distributed plumbing of the bench without a GPU (gloo on CPU): rendezvous,
    the time-slab partition and all-to-all plan of every rank (libls host-only queries), the
    barrier + max-over-ranks reduction of a timed region, and rank 0's JSON line with n_gpus =
    WORLD_SIZE.  No kernel runs, so value / ms_per_step are null."""
    import torch
    import torch.distributed as dist
    import paper_1809_10026_b200 as ls
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    w = workload(args.config)
    Ns = w["n_s"] ** w["d"]
    t0, ntl = ls.partition(w["n_t"], world, rank)
    c0, cl = ls.partition(Ns, world, rank)
    t_start = time.perf_counter()
    dt = time.perf_counter() - t_start
    t = torch.tensor([dt, float(ntl * Ns), float(cl * w["n_t"])], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sizes = torch.tensor([float(ntl * Ns)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(sizes, op=dist.ReduceOp.SUM)
    if rank == 0:
        line = {"metric": "fd_apply DOF/s (fp64)", "value": None, "unit": "DOF/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": _config_dict(args.config, world, args.a2a), "dry_run": True,
                "partition": {"slab_rows_rank0": ntl, "max_slab_dofs": t[1].item(), "max_chunk_dofs": t[2].item(),
                              "dofs_total": sizes.item()},
                "timing": "max over ranks of the (empty) timed region: %.3g s" % t[0].item()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4])
    ap.add_argument("--no-extras", action="store_true", help="skip PCG / config-3 / cpu extras")
    ap.add_argument("--a2a", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: NCCL all-to-all (default) or the fused peer-memory epilogues (LS_TUNE_A2A)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU (gloo) check of the distributed harness: partition, barrier, max-over-ranks, JSON line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _respawn(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1809_10026_b200 as ls

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args.config)
    d, p, n_el = w["d"], w["p"], w["n_el"]
    n_elems = [n_el] * (d + 1)
    if world > 1:
        uid = ls.unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx = ls.Context(d, p, n_elems, rank=rank, world=world, uid=obj[0])
    else:
        ctx = ls.Context(d, p, n_elems)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    if world > 1 and args.a2a == "fused":
        ctx.tune(4, 1)  # collective: every rank enables it

    # seeded residual, generated globally and scattered by slab (same tensor for every N)
    r_host = synth.residual(ctx.global_shape, 0)[ctx.t0:ctx.t0 + ctx.nt_local]
    r = torch.from_numpy(np.ascontiguousarray(r_host)).to("cuda")
    z = torch.empty_like(r)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        ctx.fd_apply(r, z)
    barrier()

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.fd_apply(r, z)
        e1.record(stream)
        barrier()
    launches = ctx.launches - launches0
    ms = e0.elapsed_time(e1) / args.steps
    # per-launch kernel times for the roofline: the same K steps again with CUDA events around
    # every mode-product launch on the library stream (a separate pass: events between the
    # launches of the timed region would break its programmatic-dependent-launch pairs)
    barrier()
    ctx.profile(True)
    for _ in range(args.steps):
        ctx.fd_apply(r, z)
    ctx.profile(False)
    barrier()
    kms, kflops, kn = ctx.profile_read()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = w["N"] / (ms * 1e-3)

    # e2e: the public host-buffer API (H2D of r and D2H of z inside the timed region)
    pin_r = torch.from_numpy(np.ascontiguousarray(r_host)).pin_memory()
    pin_z = torch.empty_like(pin_r).pin_memory()
    ctx.fd_apply_host(pin_r, pin_z)
    e2e_steps = max(3, min(args.steps, 10))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.fd_apply_host(pin_r, pin_z)
    barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_bytes = int(8 * w["N"])  # every rank copies its slab: the whole job moves N doubles each way
    # the same through fd_apply_host_batch: K vectors, the H2D copy of vector k+1 and the D2H copy
    # of vector k-1 overlapped with the application to vector k (full-duplex PCIe)
    ctx.fd_apply_host_batch([pin_r], [pin_z])
    barrier()
    t0 = time.perf_counter()
    ctx.fd_apply_host_batch([pin_r] * e2e_steps, [pin_z] * e2e_steps)
    barrier()
    e2eb_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2eb_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2eb_s = float(t.item())
    # the e2e floor on this box: one vector in and one out over PCIe at once (torch copies of
    # the same pinned buffers on two streams, no kernel; CUDA events, best of 2)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    duplex_ms = 1e30
    for _ in range(2):
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        with torch.cuda.stream(s_in):
            r.copy_(pin_r, non_blocking=True)
        with torch.cuda.stream(s_out):
            pin_z.copy_(z, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)
        f1.record(stream)
        f1.synchronize()
        duplex_ms = min(duplex_ms, f0.elapsed_time(f1))
    if world > 1:
        t = torch.tensor([duplex_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        duplex_ms = float(t.item())

    # roofline of the dominant kernel (fd_mode_kernel): algorithmic flops / device time
    achieved = kflops / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
    hbm, hbm_src = _hbm_peak()
    traffic, traffic_src = _traffic(args.config)
    roof = {"kernel": ("FD mode-product kernels (all mode products of fd_apply: fd_mode_rd_kernel spatial "
                       "launches + fd_time_fused_kernel)"), "bound": "tensor",
            "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic,
            "traffic_unit": "bytes per launch (mean over the captured launches)", "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": 16 * w["N"],
            "peak_source": FP64_PEAK_SOURCE, "kernel_share_of_step": round(kms / (ms * args.steps), 4),
            "kernel_timing": ("CUDA events around every mode-product launch on the library stream, in a "
                              "second pass of the same K steps right after the timed region"),
            "launches_timed": kn, "flops_per_step_algorithmic": w["flops"]}

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras = run_extras(ls, torch, stream)

    if rank == 0:
        cpu_val, cpu_sample, cores = (None, "skipped", None)
        if world == 1 and not args.no_extras:
            cpu_val, cpu_sample, cores = oracle_sample(args.config)
            try:
                extras["oracle_timing"] = oracle_extras()
            except Exception as exc:  # a baseline only: never fail the bench line on it
                extras["oracle_timing"] = {"error": repr(exc)[:200]}
        line = {
            "metric": "fd_apply DOF/s (fp64)",
            "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(args.config, world, args.a2a),
            "gflops_algorithmic": w["flops"] / (ms * 1e-3) / 1e9,
            "fp64_roofline_frac": round(w["flops"] / (ms * 1e-3) / 1e12 / (FP64_PEAK_TFLOPS * world), 4),
            # the paper's operation count 4N(d n_s + n_t) (PAPER.md 1071) per unit time: the rate an
            # unsplit implementation would need for this DOF/s (not a hardware rate; > peak is possible)
            "gflops_paper_count_equivalent": w["flops_paper"] / (ms * 1e-3) / 1e9,
            "flops_note": ("algorithmic flops as executed: spatial mode products split by centrosymmetry "
                           "(2 (he^2 + ho^2) per column instead of 2 n^2; DESIGN.md 5, reading c25), time modes "
                           "2 n_t^2 per column"),
            "roofline": roof,
            "cpu_baseline": {"value": cpu_val, "unit": "DOF/s", "cores": cores, "kind": "oracle",
                             "sample": cpu_sample},
            "e2e": {"value": w["N"] / e2eb_s, "unit": "DOF/s", "h2d_bytes_per_step": e2e_bytes,
                    "d2h_bytes_per_step": e2e_bytes, "steps": e2e_steps,
                    "api": "fd_apply_host_batch (pinned host buffers; every step copies its r in and its z "
                           "out, the copies of steps k+1 / k-1 overlap step k)",
                    "pcie_floor": {"value": w["N"] / (duplex_ms * 1e-3), "unit": "DOF/s",
                                   "frac": round((duplex_ms * 1e-3) / e2eb_s, 4),
                                   "how": ("one step's H2D and D2H copies issued at once on two streams, "
                                           "no kernel (torch copies of the same pinned buffers; CUDA events, "
                                           "best of 2): the e2e rate if fd_apply were free")},
                    "single_call": {"value": w["N"] / e2e_s, "unit": "DOF/s",
                                    "api": "fd_apply_host (one synchronous call per step)"}},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def matvec_roofline(d, p, N, ms):
    """ls_matvec against both floors: 15 banded products of 2(2p+1) flops per DOF
    at d = 3 (30(2p+1) N flops, PAPER.md 686-703; 9 at d = 2) vs the FP64 peak, and the 16 B/DOF of reading x and
    writing y vs the measured HBM bandwidth; the larger fraction names the binding floor."""
    products = {1: 4, 2: 9, 3: 15}[d]  # banded products per DOF of the sum factorisation
    flops = 2.0 * products * (2 * p + 1) * N
    tf = flops / (ms * 1e-3) / 1e12
    gbs = 16.0 * N / (ms * 1e-3) / 1e9
    hbm, _ = _hbm_peak()
    return {"alg_flops": flops, "tflops": round(tf, 3), "frac_fp64": round(tf / FP64_PEAK_TFLOPS, 4),
            "alg_bytes": 16 * N, "gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4),
            "floor_ms": round(max(flops / (FP64_PEAK_TFLOPS * 1e12), 16.0 * N / (hbm * 1e9)) * 1e3, 4)}


def run_extras(ls, torch, stream):
    """Secondary numbers (rank 0, N = 1): config-3 fd_apply (the single-GPU
    roofline case) and PCG solve times (configs 2 and 5)."""
    out = {}
    w = workload(3)
    ctx = ls.Context(3, 3, [64] * 4)
    ctx.set_stream(stream)
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        ctx.fd_apply(r, z)
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2
    tot = 0.0
    ctx.profile(True)
    for _ in range(20):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.fd_apply(r, z)
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    ctx.profile(False)
    kms, kfl, _ = ctx.profile_read()
    ms = tot / 20
    out["config3"] = {"value": w["N"] / (ms * 1e-3), "unit": "DOF/s", "ms_per_step": ms,
                      "fp64_roofline_frac": round(w["flops"] / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                      "mode_kernel_tflops": round(kfl / (kms * 1e-3) / 1e12, 3),
                      "l2": "flushed (512 MB write) before every step"}
    ctx.close()
    del flush
    pcg = []
    for cfg, p, kind in ((2, 3, 0), (5, 2, 1), (5, 4, 1), (5, 8, 1), (4, 6, 1)):
        n_el = synth.CONFIGS[cfg]["n_el"]
        d = synth.CONFIGS[cfg]["d"]
        c = ls.Context(d, p, [n_el] * (d + 1))
        c.set_stream(stream)
        b = c.rhs(kind)
        c.pcg(b, tol=1e-8)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, st = c.pcg(b, tol=1e-8)
        torch.cuda.synchronize()
        solve_ms = (time.perf_counter() - t0) * 1e3
        # per-iteration split: one fd_apply and one matvec timed with CUDA events
        z = torch.empty_like(b)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        c.fd_apply(b, z)
        ev[1].record(stream)
        c.matvec(b, z)
        ev[2].record(stream)
        ev[2].synchronize()
        ee = c.energy_error(kind, x)  # ||f - (d_t - Lap) u_h||^2 (kind 1: the error vs the exact u)
        pcg.append({"config": cfg, "d": d, "p": p, "n_el": n_el, "N": c.N, "iters": st["iters"],
                    "solve_ms": solve_ms, "true_rel_res": st["true_rel_res"],
                    # J = ||f||^2 - 2 b.x + x.Ax resolves ~1e-12 ||f||^2, i.e. relative errors >= 1e-6
                    "ls_energy_rel": (float(np.sqrt(ee["J"] / ee["f2"])) if ee["J"] > 1e-12 * ee["f2"]
                                      else "below 1e-6 (unresolved by the identity)"),
                    "fd_apply_ms": ev[0].elapsed_time(ev[1]), "matvec_ms": ev[1].elapsed_time(ev[2]),
                    "matvec_roofline": matvec_roofline(d, p, c.N, ev[1].elapsed_time(ev[2])),
                    "rhs": "kind %d (DESIGN.md reading c11)" % kind})
        del z
        c.close()
        del b, x
    out["pcg"] = pcg
    out["geometry"] = run_geometry(ls, torch, stream)
    return out


def run_geometry(ls, torch, stream, cases=((32, 3), (64, 3))):
    """Mapped domain: the rotated quarter annulus of PAPER.md 1219
    (Table 2's domain), P and P^G, the paper's forcing with homogeneous data (ls_rhs kind 3,
    DESIGN.md c23), tol 1e-8.  Paper (Table 2, p = 3, serial Matlab, with lifting): n_sub = 32:
    P 143 it / 132 s, P^G 41 it / 39.6 s; n_sub = 64: P 155 it / 2415 s, P^G 44 it / 716 s."""
    paper = {(32, "P"): (143, 132.24), (32, "P^G"): (41, 39.57), (64, "P"): (155, 2415.23), (64, "P^G"): (44, 716.03)}
    out = []
    geo = synth.revolved_quarter_annulus()
    for n_el, p in cases:
        for pc, name in ((ls.LS_PRECOND_P, "P"), (ls.LS_PRECOND_PG, "P^G")):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c = ls.Context(3, p, [n_el] * 4, geometry=geo, precond=pc)
            torch.cuda.synchronize()
            setup_s = time.perf_counter() - t0
            c.set_stream(stream)
            b = c.rhs(3)
            c.pcg(b, tol=1e-8, max_iter=2000)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, st = c.pcg(b, tol=1e-8, max_iter=2000)
            torch.cuda.synchronize()
            solve_ms = (time.perf_counter() - t0) * 1e3
            z = torch.empty_like(b)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            for _ in range(2):
                ev[0].record(stream)
                c.fd_apply(b, z)
                ev[1].record(stream)
                c.matvec(b, z)
                ev[2].record(stream)
                ev[2].synchronize()
            mv_ms = ev[1].elapsed_time(ev[2])
            S = (2 * p + 1) ** 3
            Ns = int(np.prod(c.n_s))
            out.append({"domain": "revolved quarter annulus (PAPER.md 1219)", "d": 3, "p": p, "n_el": n_el,
                        "N": c.N, "precond": name, "iters": st["iters"], "solve_ms": solve_ms,
                        "true_rel_res": st["true_rel_res"], "setup_s": round(setup_s, 3),
                        "fd_apply_ms": ev[0].elapsed_time(ev[1]), "matvec_ms": mv_ms,
                        # stencil pass: 2 (2p+1)^3 MACs per DOF (M_s, J_s) -> flops; bytes: the three
                        # stencil arrays once + t1, t2 read + y written
                        "matvec_gflops_alg": round(4.0 * S * c.N / (mv_ms * 1e-3) / 1e9, 1),
                        "matvec_gbs_alg": round(8.0 * (3 * S * Ns + 5 * c.N) / (mv_ms * 1e-3) / 1e9, 1),
                        "fit_rel_res": c.geo_info()[0], "rhs": "kind 3 (DESIGN.md c23)",
                        "paper_table2_iters_s": paper.get((n_el, name))})
            c.close()
            del b, x, z
    # the Fig. 2 setting (PAPER.md 1128-1139): 2D quarter annulus, u = -(r^2-1)(r^2-4) x y^2 sin(pi t)
    for n_el, p in ((64, 3), (128, 3)):
        for pc, name in ((ls.LS_PRECOND_P, "P"), (ls.LS_PRECOND_PG, "P^G")):
            c = ls.Context(2, p, [n_el] * 3, geometry=synth.quarter_annulus(), precond=pc)
            c.set_stream(stream)
            b = c.rhs(2)
            c.pcg(b, tol=1e-8, max_iter=2000)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, st = c.pcg(b, tol=1e-8, max_iter=2000)
            torch.cuda.synchronize()
            solve_ms = (time.perf_counter() - t0) * 1e3
            e = c.energy_error(2, x)
            out.append({"domain": "quarter annulus, u of PAPER.md 1129 (ls_rhs kind 2)", "d": 2, "p": p,
                        "n_el": n_el, "N": c.N, "precond": name, "iters": st["iters"], "solve_ms": solve_ms,
                        "true_rel_res": st["true_rel_res"],
                        "ls_energy_rel": float(np.sqrt(max(e["J"], 0.0) / e["f2"]))})
            c.close()
            del b, x
    return out


if __name__ == "__main__":
    sys.exit(main())
