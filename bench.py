"""Benchmark: BA LM-iteration time and observations/s on B200 (vs the CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c5|c4ba|c3|c1] [--no-cpu-baseline] [--no-e2e]

Workload (BASELINE.json `metric`): synthetic BA,
default C5 = 5000 cameras / 2,000,000 points / 20,000,000 observations (k=10
views per point), generate(sigma=1, seed 0) -> perturb(rot 1 deg, centre 1%,
focal 2%, point 0.5%, seed 1) -> BAProblem(Huber 1.0) -> lm_solve with the
reference's default LMConfig. A "step" is one LM iteration of that solve
(linearize + J^T r + elimination + PCG + back-substitution + candidate cost).
W warm-up iterations run first; the K timed iterations continue the same
trajectory (theta and lambda carried over) in one lm_solve call bracketed by
CUDA events on the launching stream, synchronize + barrier on both sides,
max over ranks. The working set (compact Jacobian 2 x 2.56 GB) is far larger
than the 126 MB L2, so no explicit flush is needed between iterations.

`e2e` runs the same solve through the public API from HOST numpy arrays:
problem construction (H2D copy + device ordering build), the LM iterations and
the D2H copy of theta are inside the timed region.

--impl reference times the unmodified reference package (oracle/_ref,
sparsesfm Cython/OpenMP + numpy/scipy) on the host cores on a bounded sample of
the same workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (cameras, points, visibility k, sigma, loss delta, workload label)
    "c1": (50, 5000, 4, 1.0, 1.0, "synthetic BA 50 cams / 5k pts / 20k obs (C1)"),
    "c3": (1700, 150000, 5, 1.0, 1.0, "synthetic BA 1.7k cams / 150k pts / 680k obs (C3, BAL Ladybug shape)"),
    "c4ba": (1000, 500000, 8, 1.0, 1.0, "synthetic BA 1k cams / 500k pts / 4M obs (C4 BA stage)"),
    "c5": (5000, 2000000, 10, 1.0, 1.0, "synthetic large-scale BA 5000 cams / 2M pts / 20M obs (C5)"),
    # global positioning (gp.py): rays from the observed scene, Huber 0.1, seeded init
    "c2gp": (200, 50000, 6, 0.5, 0.1, "synthetic GP 200 cams / 50k pts / 300k obs, per-observation scales (C2)"),
    "c4gp": (1000, 500000, 8, 1.0, 0.1, "synthetic GP 1k cams / 500k pts / 4M obs (C4 GP stage)"),
}
GP_CONFIGS = {"c2gp", "c4gp"}
# C4: the GP -> BA global SfM stage: GP 20 iterations (Huber 0.1)
# on the observed sigma=1 scene, then BA 10 iterations (Huber 1.0) on its output
PIPELINE = {"c4": (1000, 500000, 8, 1.0, "synthetic GP+BA global SfM 1k cams / 500k pts / 4M obs (C4)")}
# bounded CPU samples of the C5 shape for the reference, at C5's camera count
# (same k = 10 views per point): the reference's dense reduced camera system
# (40,000^2 at 5000 cameras) makes one LM iteration cost tens of seconds on the
# host whatever the point count, so the point count is what is bounded
REF_SAMPLE = (5000, 100000, 10)           # --impl reference, config c5
CPU_BASELINE_SAMPLE = (5000, 20000, 10)   # cpu_baseline leg of the b200 line
# C3: points >= 80,000 lose their highest-camera observation
C3_TRIM = 80000
METRIC = "BA/GP LM iteration time and observations/sec at 1/2/4/8 B200 vs CPU ref"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:   # the CUDA device this rank uses (CUDA_VISIBLE_DEVICES may remap indices)
            import torch
            uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:   # noqa: BLE001 - fall back to the index
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def _poll(self):
        # NVML in-process every 200 ms: no nvidia-smi process whose queries can
        # stall this process's CUDA calls (short timed regions caught 10-140 ms
        # host stalls with the subprocess sampler)
        nv, h = self.nv, self.h
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.halt.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, smax, r))
            except Exception:   # noqa: BLE001
                pass
            self.halt.wait(0.2)

    def start(self):
        self.samples, self.nv = [], None
        try:
            self.nv, self.h = self._nvml_handle()
            self.halt = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:   # noqa: BLE001 - nvidia-smi below
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.halt.set()
            self.thread.join(timeout=2)
            nv = self.nv
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            sm = [x[0] for x in self.samples]
            reasons = sorted({k for _, _, r in self.samples for k, b in bits.items() if r & b})
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self.samples[0][1] if self.samples else None,
                    "reasons": reasons, "samples": len(sm), "sampler": "nvml 200 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_arrays(cams, pts, k, sigma, seed=0, trim=None):
    from paper_2510_13310_b200 import synth
    cfg = synth.SynthConfig(num_cameras=cams, num_points=pts, visibility_fraction=k / cams,
                            pixel_noise_sigma=sigma, seed=seed)
    _, observed = synth.generate_arrays(cfg)
    arr = synth.perturb_arrays(observed, rot_deg=1.0, center_frac=0.01, focal_frac=0.02,
                               point_frac=0.005, seed=1)
    return synth.trim_points_arrays(arr, trim) if trim is not None else arr


def host_info():
    """CPU model, threads and RAM of this host"""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "threads": usable, "ram_gib": ram}


def profiled_traffic(config):
    """DRAM bytes per CG iteration of the PCG solve from the committed ncu
    capture of this config (profiles/traffic_<config>.json), or None"""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{config}.json")) as fh:
            d = json.load(fh)
        return d
    except (OSError, ValueError):
        return None


def next_lambda(cfg, rec):
    if rec.step_accepted:
        return max(rec.lam / cfg.lambda_down, cfg.lambda_min)
    return min(rec.lam * cfg.lambda_up, cfg.lambda_max)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def run_pipeline(args):
    """C4 pipeline bench (1 GPU): both stages timed with CUDA events; value =
    observations x LM iterations (both stages) / time. e2e: run_global_sfm
    from host arrays (host->device copies and the decoded scene inside)."""
    import torch
    import paper_2510_13310_b200 as b2
    from paper_2510_13310_b200 import synth
    torch.cuda.set_device(0)
    cams, pts, k, sigma, label = PIPELINE[args.config]
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=cams, num_points=pts, visibility_fraction=k / cams,
                                                     pixel_noise_sigma=sigma, seed=0))
    N = obs.num_observations
    for _ in range(max(1, args.warmup // 3)):          # warm-up: one full pipeline
        b2.run_global_sfm(obs)
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(1.0)   # nvidia-smi starts up before the timed region
    stream = torch.cuda.current_stream()
    times, gp_its, ba_its, rms, lm_ms = [], 0, 0, None, 0.0
    for _ in range(max(1, args.steps // 10)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        out, rep = b2.run_global_sfm(obs)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append((e0.elapsed_time(e1), time.perf_counter() - t0))
        gp_its += len(rep.gp.iterations)
        ba_its += len(rep.ba.iterations)
        lm_ms += sum(i.device_ms for i in rep.gp.iterations) + sum(i.device_ms for i in rep.ba.iterations)
        rms = (rep.rmse_after_gp, rep.rmse_after_ba)
    clocks = sampler.stop()
    ms = sum(t[0] for t in times)
    wall = sum(t[1] for t in times)
    its = gp_its + ba_its
    # value: the LM iterations of both stages (device time, inputs resident);
    # e2e: the whole run_global_sfm call from host arrays (setup included)
    return {"metric": METRIC, "value": N * its / (lm_ms / 1e3), "unit": "obs/s", "n_gpus": 1, "steps": its,
            "warmup": args.warmup, "ms_per_step": lm_ms / its, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "cameras": cams, "points": pts, "observations": N,
                       "stages": "GP 20 its Huber 0.1 -> BA 10 its Huber 1.0", "parallelism": "single",
                       "l2": "inputs larger than L2"},
            "pipeline_ms": round(ms / len(times), 2), "lm_ms": round(lm_ms / len(times), 2),
            "gp_iterations": gp_its, "ba_iterations": ba_its,
            "rmse_after_gp_px": rms[0], "rmse_after_ba_px": rms[1],
            "e2e": {"value": N * its / wall, "unit": "obs/s", "h2d_bytes_per_step": int(N * 40 / its),
                    "d2h_bytes_per_step": int(N * 8 / its), "note": "run_global_sfm from host arrays"},
            "clocks": clocks, "roofline": None, "gpu_launches": None}


def run_b200(args, ws, rank, local):
    import torch
    import paper_2510_13310_b200 as b2
    from paper_2510_13310_b200 import _native
    import ctypes as ct

    same_dev = ws > 1 and args.same_device
    torch.cuda.set_device(0 if same_dev else local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if same_dev:   # plumbing check of the sharded path on one GPU (not a measurement)
            os.environ["SSFM_PCG_SMS"] = str(140 // ws)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cams, pts, k, sigma, delta, label = CONFIGS[args.config]
    t0 = time.time()
    arr = make_arrays(cams, pts, k, sigma, trim=C3_TRIM if args.config == "c3" else None)
    N, P, C = arr.num_observations, arr.num_points, arr.num_cameras
    log(f"[rank {rank}] generated {label}: N={N} in {time.time() - t0:.1f}s")
    loss = b2.RobustLoss("huber", delta)
    base_cfg = b2.LMConfig()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident run (value). N > 1: points sharded over the ranks,
    # cameras replicated, camera sums exchanged through peer memory (dist.py)
    from paper_2510_13310_b200 import dist as bdist

    is_gp = args.config in GP_CONFIGS
    gp_base = b2.fix_gauge(b2.make_rays_device(arr, depth_mode=False, loss=loss, seed=0)) if is_gp else None

    def make_problem(a=None):
        a = arr if a is None else a
        if is_gp:
            return bdist.ShardedGPProblem(gp_base, rank=rank, world=ws) if ws > 1 else \
                b2.fix_gauge(b2.make_rays_device(a, depth_mode=False, loss=loss, seed=0))
        if ws > 1:
            return bdist.ShardedBAProblem(a, loss, rank=rank, world=ws)
        return b2.BAProblem(a, loss)

    def theta_start(p):
        return p.initial_theta() if is_gp else p.encode()

    problem = make_problem()
    Nl, Pl = problem.num_obs, problem.num_points
    theta0 = torch.as_tensor(theta_start(problem)).cuda()
    h = problem._native_handle()
    lib = _native.load()
    t_setup = time.time()
    # warm-up iterations (untimed)
    wcfg = b2.LMConfig(max_iterations=args.warmup)
    theta_w, rep_w = b2.lm_solve(problem, theta0, wcfg)
    lam = next_lambda(base_cfg, rep_w.iterations[-1]) if rep_w.iterations else base_cfg.lambda0
    lam = min(max(lam, base_cfg.lambda_min * 1.0000001), base_cfg.lambda_max * 0.9999999)
    log(f"[rank {rank}] warmup {len(rep_w.iterations)} its {time.time() - t_setup:.1f}s, lambda -> {lam:g}")
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(1.0)   # nvidia-smi starts up before the timed region
    stream = torch.cuda.current_stream()
    # exactly K timed LM iterations: continue the warm-up trajectory; if a
    # solve converges early, the next one restarts from theta0 (same workload)
    ms_total, steps, iters = 0.0, 0, []
    pms_sum, pl_sum, cg_sum, launch_sum = 0.0, 0, 0.0, 0
    phase_sum = [0.0] * 5
    # theta stays resident in HBM across the timed region (CUDA tensors in,
    # CUDA tensors out): no host copies inside it
    dev_theta = lambda t: t if isinstance(t, torch.Tensor) else torch.as_tensor(np.asarray(t), device="cuda")  # noqa: E731
    theta0_dev = dev_theta(theta0)
    theta_cur, lam_cur = dev_theta(theta_w), lam
    torch.cuda.synchronize()
    barrier()
    while steps < args.steps:
        tcfg = b2.LMConfig(max_iterations=args.steps - steps, lambda0=lam_cur)
        lib.ssfm_profile_enable(ct.c_void_p(h.ptr), 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        theta_t, rep_t = b2.lm_solve(problem, theta_cur, tcfg)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_total += e0.elapsed_time(e1)
        pms, pl, cgit = ct.c_double(0), ct.c_int64(0), ct.c_double(0)
        lib.ssfm_profile_get(ct.c_void_p(h.ptr), 0, ct.byref(pms), ct.byref(pl), ct.byref(cgit))
        ams, launches, _ = ct.c_double(0), ct.c_int64(0), ct.c_double(0)
        lib.ssfm_profile_get(ct.c_void_p(h.ptr), 2, ct.byref(ams), ct.byref(launches), ct.byref(_))
        pms_sum += pms.value; pl_sum += pl.value; cg_sum += cgit.value; launch_sum += launches.value
        for kk in range(5):
            phm = ct.c_double(0)
            lib.ssfm_profile_get(ct.c_void_p(h.ptr), 3 + kk, ct.byref(phm), None, None)
            phase_sum[kk] += phm.value
        iters += rep_t.iterations
        steps += len(rep_t.iterations)
        if rep_t.termination != "max_iter" or not rep_t.iterations:
            theta_cur, lam_cur = theta0_dev, base_cfg.lambda0
        else:
            theta_cur = theta_t
            lam_cur = min(max(next_lambda(base_cfg, rep_t.iterations[-1]), base_cfg.lambda_min * 1.0000001),
                          base_cfg.lambda_max * 0.9999999)
    barrier()
    clocks = sampler.stop()
    lib.ssfm_profile_enable(ct.c_void_p(h.ptr), 0)
    pms, pl, cgit = ct.c_double(pms_sum), ct.c_int64(pl_sum), ct.c_double(cg_sum)
    launches = ct.c_int64(launch_sum)
    rep_t.iterations = iters
    ms_max = ms_total
    if dist is not None:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    ms_per_step = ms_max / max(steps, 1)
    value = N * steps / (ms_max / 1e3)
    log(f"[rank {rank}] timed {steps} its in {ms_total:.1f} ms; cg {[i.cg_iters for i in rep_t.iterations]}; "
        f"term {rep_t.termination}; device ms {[round(i.device_ms, 2) for i in rep_t.iterations]}")

    # roofline of the dominant kernel: the PCG solve (ba_k_pcg), S*p dominated
    peak, peak_kind = peaks()
    # SURVEY.md 8(d), S*p per CG iteration (this rank)
    bytes_per_cg = (40.0 * Nl + 72.0 * Pl + 48.0 * C) if is_gp else (136.0 * Nl + 72.0 * Pl + 128.0 * C)
    roof = None
    if pms.value > 0 and cgit.value > 0:
        ach = bytes_per_cg * cgit.value / (pms.value / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": None, "peak_source": peak_kind,
                "kernel": "GP PCG solve (CUDA graph or gp_k_pcg)" if is_gp else "BA PCG solve (CUDA graph or ba_k_pcg)", "launches": int(pl.value),
                "cg_iters": int(cgit.value),
                "kernel_ms": round(pms.value, 3),
                "algorithmic_bytes_per_cg_iter": bytes_per_cg,
                "kernel_share_of_step": round(pms.value / max(ms_total, 1e-9), 4)}
        prof = profiled_traffic(args.config) if ws == 1 else None
        if prof is not None:
            # ncu dram__bytes_read.sum + dram__bytes_write.sum of the PCG's
            # kernels per CG iteration (profiles/traffic_<config>.json)
            roof["traffic"] = prof["dram_bytes_per_cg_iter"]
            roof["traffic_unit"] = "bytes per CG iteration (ncu, all PCG kernels)"
            roof["traffic_over_algorithmic"] = round(prof["dram_bytes_per_cg_iter"] / bytes_per_cg, 3)
            roof["traffic_source"] = prof.get("source")
        if not is_gp and sum(phase_sum) > 0:
            names = ["point_or_fused_pass", "camera_pass", "q_and_pq", "x_r_z_update", "p_update"]
            roof["phase_ms_per_cg_iter"] = {n: round(v / cgit.value, 4) for n, v in zip(names, phase_sum)}
    del theta_t

    # ---- end to end through the public API from host arrays
    e2e = None
    if not args.no_e2e:
        theta_host = theta_start(problem)
        # the per-observation inputs live in pinned host memory (staged before
        # the timed region, as an application feeding the solver would)
        def pinned(x):
            t = torch.empty(x.shape, dtype=getattr(torch, str(x.dtype)), pin_memory=True)
            t.numpy()[...] = x
            return t.numpy()
        arr_host = arr.copy()
        arr_host.cam_idx, arr_host.pt_idx, arr_host.pixels = (pinned(np.asarray(arr.cam_idx)),
                                                             pinned(np.asarray(arr.pt_idx)),
                                                             pinned(np.asarray(arr.pixels)))
        theta_host = pinned(np.asarray(theta_host))

        def one_e2e(tag):
            barrier()
            t_a = time.perf_counter()
            e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_a.record(stream)
            p2 = make_problem(arr_host)
            t_c = time.perf_counter()
            th_out, rep_e = b2.lm_solve(p2, theta_host, b2.LMConfig(max_iterations=args.warmup + args.steps))
            t_s = time.perf_counter()
            e_b.record(stream)
            barrier()
            wall = time.perf_counter() - t_a
            e_ms = e_a.elapsed_time(e_b)
            log(f"[rank {rank}] e2e ({tag}): problem + handle {1e3 * (t_c - t_a):.0f} ms, lm_solve "
                f"{1e3 * (t_s - t_c):.0f} ms ({len(rep_e.iterations)} its, device "
                f"{sum(i.device_ms for i in rep_e.iterations):.0f} ms)")
            its = max(len(rep_e.iterations), 1)
            if dist is not None:
                t = torch.tensor([wall], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                wall = float(t.item())
            # bytes moved host -> device: the per-observation inputs as stored on
            # the host (indices narrowed to int32 on the device), camera
            # intrinsics, theta; device -> host: theta
            h2d = (Nl * (np.asarray(arr_host.cam_idx).itemsize + np.asarray(arr_host.pt_idx).itemsize
                         + (24 if is_gp else 16)) + C * (16 + 16 + 8) + theta_host.nbytes)
            out = {"value": N * its / wall, "unit": "obs/s",
                   "first_iteration_ms": round(rep_e.iterations[0].device_ms, 3) if rep_e.iterations else None,
                   "time_to_solution_s": round(wall, 3), "setup_ms": round(1e3 * (t_c - t_a), 1),
                   "h2d_bytes_per_step": int(h2d / its), "d2h_bytes_per_step": int(theta_host.nbytes / its),
                   "iterations": its, "wall_s": round(wall, 3), "device_ms": round(e_ms, 1),
                   "termination": rep_e.termination}
            return out, p2

        # cold: the device-timed handle is destroyed and the library's block
        # cache emptied, so problem creation allocates HBM from scratch (an
        # application's first solve). warm: the same solve again after that
        # handle is released into the cache (an application solving problems of
        # one shape in turn: creation skips cudaMalloc)
        if ws == 1 and hasattr(problem, "release"):
            problem.release(trim=True)
        e2e, p2 = one_e2e("cold")
        if ws == 1 and hasattr(p2, "release"):
            p2.release()
        del p2
        warm, p3 = one_e2e("warm")
        del p3
        e2e["cache"] = "cold (no reused device blocks)"
        e2e["warm"] = {k: warm[k] for k in ("value", "time_to_solution_s", "setup_ms", "device_ms")}
    result = {
        "metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": ws, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "cameras": C, "points": P, "observations": N,
                   "views_per_point": k, "loss": f"huber({delta})", "lm": "LMConfig() defaults",
                   "problem": "gp" if is_gp else "ba",
                   "parallelism": f"points sharded over {ws} GPUs" if ws > 1 else "single",
                   "observations_per_rank": Nl,
                   "l2": "inputs larger than L2 (J 2x2.56 GB)" if N >= 10**6 else "small (latency bound)"},
        "cg_iters_per_step": [i.cg_iters for i in rep_t.iterations],
        "lm_ms_per_iteration": [round(i.device_ms, 3) for i in rep_t.iterations],
        # LM-iteration time = median over iterations 2..n; the
        # first iteration of a solve (setup, first linearization) separately
        "lm_ms_median": round(statistics.median([i.device_ms for i in rep_t.iterations[1:]]
                                                or [i.device_ms for i in rep_t.iterations]), 3),
        "roofline": roof, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches.value),
    }
    if rank == 0 and not args.no_cpu_baseline and not is_gp:
        result["cpu_baseline"] = cpu_baseline_sample(max_iterations=2)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return result


# ---------------------------------------------------------------------------
# reference (CPU) side
# ---------------------------------------------------------------------------
def _import_reference():
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "sparsesfm")):
        return None, f"reference not built ({ref_dir}); run oracle/build_ref.sh"
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    os.environ.setdefault("SPARSESFM_BACKEND", "cython")
    ncpu = os.cpu_count() or 1
    os.environ.setdefault("SPARSESFM_WORKERS", str(ncpu))
    import sparsesfm
    return sparsesfm, None


def cpu_baseline_sample(max_iterations=2):
    """Bounded sample: the reference on a C5-shaped reduction at C5's camera
    count (k = 10); value from the iterations after the first (which includes
    the pattern build)."""
    ref, why = _import_reference()
    if ref is None:
        return {"value": None, "unit": "obs/s", "cores": 0, "kind": "reference", "sample": why}
    from sparsesfm import synth_metrics as rsm
    cams, pts, k = CPU_BASELINE_SAMPLE
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=cams, num_points=pts,
                                              visibility_fraction=k / cams, pixel_noise_sigma=1.0, seed=0))
    start = rsm.perturb(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    prob = ref.BAProblem(start, ref.RobustLoss("huber", 1.0))
    t0 = time.perf_counter()
    _, rep = ref.lm_solve(prob, prob.encode(), ref.LMConfig(max_iterations=max_iterations))
    wall = time.perf_counter() - t0
    its = rep.iterations
    later = [i.wall_time_ns for i in its[1:]] or [i.wall_time_ns for i in its]
    med = statistics.median(later) / 1e9
    n = start.num_observations
    return {"value": n / med, "unit": "obs/s", "cores": int(os.environ.get("SPARSESFM_WORKERS", "1")),
            "kind": "reference",
            "sample": f"reference sparsesfm (Cython/OpenMP backend) BA {cams} cams / {pts} pts / {n} obs "
                      f"(C5 shape, k={k}), {len(its)} LM iterations, median of iterations 2..n "
                      f"({med:.2f} s/iter; first {its[0].wall_time_ns / 1e9:.2f} s incl. pattern build); "
                      f"total {wall:.1f} s",
            "s_per_iter_median": med, "host": host_info()}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    ref, why = _import_reference()
    if ref is None:
        return {"impl": "reference", "unavailable": why}
    if args.config in PIPELINE:
        return {"impl": "reference", "unavailable": "the reference has no GP->BA pipeline function "
                "(SURVEY.md 8(d) C4); its stages are timed by --config c4gp / c4ba"}
    cams, pts, k, sigma, delta, label = CONFIGS[args.config]
    from sparsesfm import synth_metrics as rsm
    is_gp = args.config in GP_CONFIGS
    # bounded samples keep the CPU run to a few minutes: C5 (does not fit /
    # ~2 min per iteration) and the 4M-observation GP stage
    scams, spts, sk = REF_SAMPLE if args.config == "c5" else \
        ((1000, 50000, 8) if args.config == "c4gp" else (cams, pts, k))
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=scams, num_points=spts,
                                              visibility_fraction=sk / scams, pixel_noise_sigma=sigma,
                                              seed=0))
    if is_gp:
        prob = ref.fix_gauge(ref.make_rays(obs, False, ref.RobustLoss("huber", delta), seed=0))
        th0 = prob.initial_theta()
        n = obs.num_observations
    else:
        start = rsm.perturb(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
        if args.config == "c3":     # the same trimmed 680k-observation recipe as the b200 arm
            top = {}
            for o in start.observations:
                top[o.point_id] = max(top.get(o.point_id, -1), o.camera_id)
            start = ref.Scene(start.cameras, start.points,
                              [o for o in start.observations
                               if not (o.point_id >= C3_TRIM and o.camera_id == top[o.point_id])])
        prob = ref.BAProblem(start, ref.RobustLoss("huber", delta))
        th0 = prob.encode()
        n = start.num_observations
    cfg = ref.LMConfig(max_iterations=args.warmup + args.steps)
    t0 = time.perf_counter()
    _, rep = ref.lm_solve(prob, th0, cfg)
    wall = time.perf_counter() - t0
    its = rep.iterations
    timed = its[args.warmup:] or its
    t_timed = sum(i.wall_time_ns for i in timed) / 1e9
    value = n * len(timed) / t_timed
    cores = int(os.environ.get("SPARSESFM_WORKERS", "1"))
    bounded = args.config in ("c5", "c4gp")
    sample = (f"reference sparsesfm {'GP' if is_gp else 'BA'} {scams} cams / {spts} pts / {n} obs (k={sk}"
              f"{', bounded sample of the config shape' if bounded else ''}); "
              f"{len(its)} LM iterations, last {len(timed)} timed; total {wall:.1f} s")
    return {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": ws, "steps": len(timed),
            "warmup": args.warmup, "ms_per_step": 1e3 * t_timed / len(timed), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "sample_cameras": scams, "sample_points": spts,
                       "sample_observations": n},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "obs/s", "cores": cores, "kind": "reference",
                             "sample": sample, "host": host_info(),
                             "s_per_iter": [round(i.wall_time_ns / 1e9, 3) for i in its]},
            "e2e": {"value": value, "unit": "obs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "termination": rep.termination}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS) + sorted(PIPELINE))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--same-device", action="store_true",
                    help="N>1 ranks all on cuda:0 over gloo: plumbing check of the sharded path, not a measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    ws, rank, local = dist_env()
    if args.impl == "reference":
        res = run_reference(args, ws, rank)
    elif args.config in PIPELINE:
        res = run_pipeline(args) if rank == 0 else None
    else:
        res = run_b200(args, ws, rank, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
