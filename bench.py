#!/usr/bin/env python
"""Benchmark of the GMAF hot path on B200 (contract: see DESIGN.md sec. 8).

One *step* = one joint Picard-step analysis of K working conditions through the
public API (gmaf_thickness -> gmaf_assemble -> gmaf_solve(rtol) -> gmaf_integrate),
i.e. every row of SURVEY 8(a), on BASELINE config C3 by default (short-textured
2048x1024, K = 9, omega 1.6, rtol 1e-10).

metric  = PCG-ASSOR DOF*iter/s = sum_steps K*n_theta*n_y*iterations / device time.
value   : CUDA-event time over the timed steps (inputs -- the K condition records --
          are re-sent every step; the fields are HBM-resident, 151 MB each > L2).
e2e     : the same steps timed on the host clock, H2D of the condition records and D2H
          of the wrench and solve statistics inside.
roofline: the dominant kernel's algorithmic bytes / its measured average duration
          (in-kernel %globaltimer over the timed region), against MEASURED_PEAKS.json.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl gmaf|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gmaf_inputs as gi  # noqa: E402

METRIC = "PCG-ASSOR DOF*iter/s (joint K-condition solve, full Picard-step analysis)"
UNIT = "DOF*iter/s"


def _ncu_traffic(kernel: str, cfg_name: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
    kernel from the committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tab = json.load(f)
        ent = tab.get(f"{cfg_name}:{kernel}")
        return None if ent is None else float(ent["dram_bytes_per_launch"])
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _host_info() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def _full_step_iterations(cfg) -> int | None:
    """PCG iterations of one full step of this workload as the ORACLE counts them (its own Table-1
    solve, tests/golden/<cfg>_oracle_samples.json, written by scripts/oracle_c3_reference.py)."""
    path = os.path.join(ROOT, "tests", "golden", f"{cfg.name.lower()}_oracle_samples.json")
    try:
        with open(path) as f:
            return int(json.load(f)["iterations"])
    except Exception:
        return None


def _oracle_sample(cfg, iters: int):
    """Time the oracle as it stands, pinned to ONE host core (sched_setaffinity = taskset -c 0;
    the oracle is single-threaded): assembly of all K conditions, `iters` PCG-ASSOR iterations,
    the K wrench quadratures."""
    import oracle
    oracle.build()
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    pinned = False
    try:
        if old is not None:
            os.sched_setaffinity(0, {min(old)})
            pinned = True
        t0 = time.perf_counter()
        AP, AE, AN, S = oracle.assemble_joint(cfg.grid, cfg.conds)
        t1 = time.perf_counter()
        res = oracle.pcg_joint(AP, AE, AN, S, tol=0.0, omega=cfg.omega, max_iter=iters)
        t2 = time.perf_counter()
        for k in range(cfg.K):
            oracle.wrench(cfg.grid, cfg.conds[k], res.p[k])
        t3 = time.perf_counter()
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return {"assembly_s": t1 - t0, "iter_s": (t2 - t1) / max(res.iterations, 1), "quadrature_s": t3 - t2,
            "iterations": res.iterations, "core": min(old) if pinned else None}


def _full_step_rate(cfg, smp) -> tuple[float, float, int | None]:
    """(full-step rate, per-iteration rate, I): the oracle's rate for the SAME workload the GPU arm
    times -- a full step with I PCG iterations (the oracle's own count) -- from the timed pieces:
    K n I / (t_assembly + t_quadrature + I t_iteration); the per-iteration rate beside it."""
    n = cfg.grid["n_theta"] * cfg.grid["n_y"]
    it_rate = cfg.K * n / smp["iter_s"]
    I = _full_step_iterations(cfg)
    if I is None:
        return it_rate, it_rate, None
    return cfg.K * n * I / (smp["assembly_s"] + smp["quadrature_s"] + I * smp["iter_s"]), it_rate, I


def cpu_baseline(cfg, iters: int = 10):
    """The oracle as it stands (single-threaded C, one core), on a bounded sample of the same
    workload: assembly of all K conditions + `iters` PCG-ASSOR iterations + the quadrature."""
    smp = _oracle_sample(cfg, iters)
    value, it_rate, I = _full_step_rate(cfg, smp)
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{cfg.name}: oracle on 1 host core (affinity core {smp['core']}, like taskset -c "
                      f"{smp['core']}): assembly of K={cfg.K} ({smp['assembly_s']:.2f} s) + {smp['iterations']} "
                      f"PCG-ASSOR iterations ({smp['iter_s'] * smp['iterations']:.2f} s) + K quadratures "
                      f"({smp['quadrature_s']:.2f} s); value = the full step of {I} iterations (the oracle's own "
                      f"count, tests/golden) from these pieces",
            "per_iteration_rate": it_rate, "full_step_iterations": I,
            "assembly_s": smp["assembly_s"], "iter_s": smp["iter_s"], "quadrature_s": smp["quadrature_s"],
            **_host_info()}


def run_reference(args, cfg):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    iters = args.ref_iters
    vals, its, steps_s = [], [], []
    last = None
    for s in range(args.warmup + args.steps):
        smp = _oracle_sample(cfg, iters)
        if s >= args.warmup:
            v, itr, I = _full_step_rate(cfg, smp)
            vals.append(v)
            its.append(itr)
            steps_s.append(smp["assembly_s"] + smp["quadrature_s"] + (I or iters) * smp["iter_s"])
            last = (smp, I)
    value = len(vals) / sum(1.0 / v for v in vals)          # the rate of the summed (equal-work) steps
    smp, I = last
    how = (f"value = the full step of {I} iterations (the oracle's own count, tests/golden) from the timed pieces"
           if I else "value = the per-iteration rate of the sample (no oracle full-step count for this config)")
    sample = (f"{cfg.name}: per step the oracle (1 host core, affinity core {smp['core']}) assembles K={cfg.K}, "
              f"runs {iters} PCG-ASSOR iterations and integrates K wrenches; {how}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(steps_s) / len(steps_s),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_obj(cfg, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "per_iteration_rate": statistics.mean(its), "full_step_iterations": I,
                             **_host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config_obj(cfg, args):
    g = cfg.grid
    return {"workload": f"{cfg.name}: {cfg.note}, omega {cfg.omega}, rtol {cfg.tol:g}, ASSOR-II, "
                        "coupled synchronized convergence (Eq. 3.9)",
            "n_theta": g["n_theta"], "n_y": g["n_y"], "K": cfg.K,
            "texture": "short 60x10" if g.get("tex_n_theta") else "smooth",
            "dof": cfg.dof,
            "l2_policy": (f"inputs larger than L2 ({cfg.dof * 8 / 1e6:.0f} MB per field, 126 MB L2)"
                          if cfg.dof * 8 > 126e6 else
                          f"working set L2-resident ({cfg.dof * 8 / 1e6:.1f} MB per field): not an HBM measurement"),
            "parallelism": "1 GPU" if args.gpus == 1 and not args.partition else
            f"{args.gpus} GPU(s): the {cfg.K}-condition joint system split into {args.gpus} row slabs (all "
            f"{cfg.K} conditions per GPU); per PCG iteration the 4 boundary rows of r and of the search "
            f"direction are stored into the neighbours' inboxes over NVLink peer memory and one gather of the "
            f"per-condition sums is summed in rank order, inside the solve's CUDA graph (strong)"
            if _partition(args) == "rows" else
            f"{args.gpus} GPUs: one joint system of {cfg.K}x{args.gpus} conditions, condition-sharded "
            f"({cfg.K} per GPU); per PCG iteration one gather of the per-condition sums "
            f"({os.environ.get('GMAF_DIST', 'p2p')}: "
            f"{'NCCL allgather' if os.environ.get('GMAF_DIST', 'p2p') == 'nccl' else 'fused into the iteration kernel over NVLink peer memory'}) (weak)"}


def picard_steps(device: int, n_steps: int) -> dict:
    """The metric's "ms per Picard step" (BASELINE.json): full time steps of the
    Picard march (Sec. 2.3) on C4's mesh -- short-textured 1024x512, each Picard iteration one
    joint 9-condition thickness -> assembly -> PCG-ASSOR-II -> quadrature on the device plus the
    host update (generalized forces, FD Jacobians, 4x4 solve; R-A28..A31) -- 1-degree steps from
    phi = 0, warm-started solves.  Host wall clock (the update runs on the host between solves)."""
    import math
    import paper_2511_06824_b200 as P
    g = gi.grid(1024, 512, "short")
    pump = gi.pump()
    dt = 2 * math.pi / gi.OMEGA_S / 360.0
    S = P.JointSolver(g, 9, device=device)
    state = gi.condition(phi_deg=0.0, p_in=gi.p_in_trapezoid(0.0))

    def step(s):
        nonlocal state
        phi = s * math.pi / 180.0
        st = state.copy()
        st[8:13] = [gi.coupling_length(phi), 0.0, gi.stroke_speed(phi), gi.p_in_trapezoid(phi), gi.P_OUT]
        state, n_pic, res, pcg, code = S.picard_step(pump, st, phi, dt, "general", eps_dyn=1e-3, max_picard=20,
                                                     tol=1e-10, omega=1.6, raise_on_error=False)
        return n_pic, pcg, code

    step(1)                                          # warm-up step (graph instantiation)
    t0 = time.perf_counter()
    rows = [step(s) for s in range(2, 2 + n_steps)]
    ms = (time.perf_counter() - t0) * 1e3
    S.close()
    n_pic = sum(r[0] for r in rows)
    return {"config": "C4 mesh: short-textured 1024x512, K=9 per Picard iteration, general scheme, "
                      "eps_dyn 1e-3, 1-degree time steps from phi=0 (warm-up step 1, timed steps 2..)",
            "time_steps": n_steps, "ms_per_time_step": ms / n_steps,
            "ms_per_picard_iteration": ms / max(n_pic, 1), "picard_iterations": [r[0] for r in rows],
            "pcg_iterations_per_step": [r[1] for r in rows], "status": [r[2] for r in rows],
            "timing": "host wall clock (device solves + host update)",
            "full_trajectory": "profiles/round1_picard_3rev_c4.json (1080 steps, 527 s)"}


def _partition(args) -> str:
    """N > 1: row slabs of the one K-condition system (default; SURVEY 8(e) for C3, strong
    scaling) or one joint system of K*N conditions, condition-sharded (C5 layout, weak)."""
    if args.partition:
        return args.partition
    return "rows" if args.gpus > 1 else "none"


def run_gmaf(args, cfg):
    import torch
    world, rank, local = _dist()
    # plumbing check on a one-GPU box (tests only): every rank on cuda:0, gloo for the host
    # collectives (NCCL refuses two ranks on one GPU); the device path is the same
    same_dev = os.environ.get("GMAF_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("gloo" if same_dev else "nccl")
        dist = tdist
    import paper_2511_06824_b200 as P
    P.lib()
    K, n = cfg.K, cfg.grid["n_theta"] * cfg.grid["n_y"]
    # N GPUs (weak scaling, C5-style): ONE joint system of 9*N conditions -- operating point r
    # (shaft angle 90 + r deg) and its 8 FD perturbations on rank r -- condition-sharded with one
    # NCCL allgather of the packed dot products per iteration (synchronized convergence, Eq. 3.9)
    from paper_2511_06824_b200.dist import aggregate, operating_point_of
    part = _partition(args) if not args.shard else "conditions"
    n_local = n
    if part == "rows":
        # row slabs: every rank holds all K conditions on its own rows; halo rows and the
        # per-condition sums are exchanged over peer memory inside the solve's CUDA graph
        S = P.JointSolver(cfg.grid, K, device=local, rank=rank, world=world, shard="rows")
        if dist:
            from paper_2511_06824_b200.dist import connect_p2p
            connect_p2p(S)
        else:
            S.p2p_connect([S.p2p_handle()])
        conds = cfg.conds
        n_local = cfg.grid["n_theta"] * (S.slab[1] - S.slab[0])
    elif world > 1 or part == "conditions":
        conds_all = np.concatenate([cfg.conds if r == 0 else
                                    gi.fd_conditions(gi.condition(phi_deg=operating_point_of(r)))
                                    for r in range(world)])
        if os.environ.get("GMAF_DIST", "p2p") == "nccl":
            # NCCL mode: one ncclAllGather + a scalar kernel per iteration, host-polled batches
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(P.gmaf_nccl_unique_id()), dtype=torch.uint8))
            if dist:
                dist.broadcast(uid, 0)
            S = P.JointSolver(cfg.grid, K * world, device=local, rank=rank, world=world,
                              nccl_uid=bytes(uid.cpu().numpy().tobytes()))
        else:
            # peer-to-peer mode (default): the per-iteration gather is fused into the iteration
            # kernel over IPC-mapped peer memory (NVLink); one CUDA graph per solve
            S = P.JointSolver(cfg.grid, K * world, device=local, rank=rank, world=world, p2p=True)
            if dist:
                from paper_2511_06824_b200.dist import connect_p2p
                connect_p2p(S)
            else:
                S.p2p_connect([S.p2p_handle()])
        conds = conds_all
    else:
        conds = cfg.conds
        # the FD conditions of Eqs. 2.17-2.19 need 5 distinct coefficient sets per 9 (Eq. 2.3 has
        # no e-dot): the band storage is sized for exactly that
        S = P.JointSolver(cfg.grid, K, device=local, max_matrices=5 * (K // 9) if K % 9 == 0 else None)
    stream = S.stream

    def one_step():
        st, W = S.step(conds, tol=cfg.tol, omega=cfg.omega, precond="assor2")
        return st

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    S.reset_kernel_times()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    iters = []
    w0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.steps):
        st = one_step()
        iters.append(st.iterations)
    ev1.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    ck = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)
    wall_ms = (w1 - w0) * 1e3
    kt = S.kernel_times()
    if dist:
        dist.barrier()
    agg = aggregate(dev_ms, wall_ms, float(K * n_local * sum(iters)),
                    device="cpu" if same_dev else "cuda")   # local DOF
    dev_max_ms, wall_max_ms, total_dof_iters = agg.device_ms_max, agg.wall_ms_max, agg.dof_iters_total
    value = agg.rate()
    e2e_value = agg.e2e_rate()

    # roofline of the dominant kernel.  Its average duration is taken two ways over the timed
    # region: (a) CUDA events around the steps minus the other kernels' device time, divided by
    # the number of launches (conservative: includes launch gaps); (b) in-kernel %globaltimer.
    dom = max((k for k in kt if k["launches"] > 0), key=lambda k: k["total_ms"])
    other_ms = sum(k["total_ms"] for k in kt if k is not dom and not k["name"].startswith("tail_"))
    avg_ev_s = max(dev_ms - other_ms, 1e-9) * 1e-3 / dom["launches"]
    avg_gt_s = dom["total_ms"] * 1e-3 / dom["launches"]
    achieved = dom["bytes_per_launch"] / avg_ev_s / 1e9
    peak, peak_src = _peaks()
    traffic = _ncu_traffic(dom["name"], cfg.name)
    solve_ms = sum(k["total_ms"] for k in kt if k["name"].startswith(("pcg_", "sr_", "true_")))
    # kernels this process launched in the timed region: every timed kernel's launches, except that
    # the persistent solve runs ALL its iterations ("sr_iter" entries, one per PCG iteration) in one
    # k_srp launch, followed by one fix-up launch (untimed); tails and barrier waits are not launches
    tiles = S.tile_config()
    persistent = bool(tiles["persistent"])
    n_solves = args.steps
    launches = int(sum(k["launches"] for k in kt
                       if not k["name"].startswith(("tail_", "gridbar_")) and not (persistent and k["name"] == "sr_iter")))
    launches += (2 * n_solves) if persistent else n_solves   # k_srp + k_sr_fixup, or the fix-up alone
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if part == "rows" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config_obj(cfg, args),
        "iterations_per_step": iters,
        "roofline": {"bound": "hbm", "kernel": dom["name"], "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)",
                     "bytes_per_launch": dom["bytes_per_launch"],
                     "avg_launch_us_events": avg_ev_s * 1e6, "avg_launch_us_globaltimer": avg_gt_s * 1e6,
                     "achieved_globaltimer": dom["bytes_per_launch"] / avg_gt_s / 1e9,
                     "canonical_equiv_frac": value / max(world, 1) * 120.0 / (peak * 1e9),
                     "unit_of_launch": ("one PCG iteration of the persistent kernel k_srp (all iterations of a "
                                        "solve run in one cooperative launch)") if persistent else
                                       "one launch of the per-iteration kernel k_sr",
                     "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the iteration kernel per "
                                     "PCG iteration (profiles/ncu_traffic.json), the same unit as bytes_per_launch",
                     "note": "achieved = algorithmic bytes (DESIGN.md sec. 6) / event-timed launch; "
                             "canonical_equiv_frac = per-GPU DOF*iter/s x 120 B (SURVEY 8(d) S1 3-band) / peak"},
        "kernels": {k["name"]: {"launches": k["launches"], "total_ms": round(k["total_ms"], 3),
                                "avg_us": round(1e3 * k["total_ms"] / k["launches"], 2) if k["launches"] else 0,
                                "GBps": round(k["bytes_per_launch"] * k["launches"] / (k["total_ms"] * 1e-3) / 1e9, 1)
                                if k["launches"] and k["total_ms"] > 0 else 0}
                    for k in kt},
        "solve_kernel_share_of_step": solve_ms / dev_ms if dev_ms else None,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": K * 13 * 8 + 48,
                "d2h_bytes_per_step": K * 12 * 8 + 8 * 7 * K + 128},
        "gpu_launches": launches,
        "tiles": tiles,
        "clocks": ck,
    }
    if rank == 0 and world == 1 and args.picard_steps > 0:
        line["picard"] = picard_steps(local, args.picard_steps)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, iters=args.ref_iters)
    if rank == 0:
        print(json.dumps(line), flush=True)
    S.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="gmaf", choices=["gmaf", "reference"])
    ap.add_argument("--ref-iters", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="use the condition-sharded path even on one GPU (1-rank communicator)")
    ap.add_argument("--picard-steps", type=int, default=3,
                    help="time C4 Picard time steps after the main measurement (0: skip; 1 GPU only)")
    ap.add_argument("--partition", choices=["rows", "conditions"], default=None,
                    help="N > 1: row slabs of the K-condition system (default, strong scaling) or a "
                         "K*N-condition system sharded by conditions (weak); also valid on 1 GPU")
    args = ap.parse_args()
    cfg = gi.config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_gmaf(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
