"""bench.py — retained Θ entries/s of the exact product-convolution wavelet decomposition on B200.

Workload: BASELINE.json config 5 (2-D 1024², Daubechies-4, J=8, m=10, band rule L=128 per unit,
fp32) — synthetic seeded inputs of synth/configs.py (there is no dataset in the paper's path).
One step = one pcwd_decompose over all units (templates a1, fused k-sum + windowed cascade +
band gather a2-a4) with u, v already resident in HBM.  L2 is flushed (256 MiB write) before
every timed step, outside the event pair.

  python bench.py [--gpus N --steps K --warmup W --config c5 --impl ours|reference]
  (N > 1: one rank per GPU — launched by torchrun, or re-launched under it by this script when WORLD_SIZE is
  unset; units sharded by cost, no collective on the data path; per step a barrier, then the max over ranks)
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

WORKLOAD = {"c5": "2-D torus 1024x1024, Daubechies-4, J=8, m=10, band L=128 per unit, fp32",
            "c3": "2-D torus 256x256, Daubechies-4, J=6, m=8, band L=64 per unit, fp32"}
METRIC = "retained Theta entries/sec (decomposition)"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self._p:
            self._p.terminate()
            try:
                self._p.wait(timeout=2)
            except Exception:
                self._p.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, val in zip(names, s[4:8]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def _ncu_traffic(kind: str, level: int):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest committed `ncu --set full`
    raw page (profiles/*/ncu_raw_fine_level{level}_*.csv), or None."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_raw_{kind}_level{level}_*.csv")))
    if not files:
        return None, None
    rows = list(csv.reader(open(files[-1])))
    if len(rows) < 3:
        return None, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if name not in rows[0]:
            return None, None
        i = rows[0].index(name)
        tot += float(rows[2][i].replace(",", "")) * scale.get(rows[1][i], 1.0)
    return tot, os.path.relpath(files[-1], ROOT)


def relaunch_under_torchrun(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-run this command as N ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1 and return its exit code; None when already a rank (or N = 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_rate(p, budget_s: float = 20.0, seed: int = 0):
    """Oracle (oracle/rows.c + brute-force band ranking) timed on a bounded stratified sample of units.

    Levels are measured finest first (one unit per host thread, one batch per level) while the running time
    stays within `budget_s`; a level whose single unit would exceed what is left is not run.  The oracle's
    per-unit cost is dominated by the adjoint sum over the nonzeros of ψ_μ (rows.c), so unmeasured levels are
    extrapolated with t(ℓ) = a + b·|supp ψ_ℓ| fitted (least squares) on the measured levels.  entries/s =
    nnz / Σ_ℓ count(ℓ)·t(ℓ)."""
    from oracle import basis
    from oracle import retention as ret
    from oracle import rows as R
    rng = np.random.default_rng(seed)
    nthreads = os.cpu_count() or 1
    levels = {}
    for (lev, e, off, nl) in basis.subbands(p.d, p.n, p.J):
        levels.setdefault(lev, []).append((off, nl ** p.d))
    lev_order = sorted(levels)

    def supp(lev):   # nonzeros of ψ_μ at level ℓ (P:103-104 length, periodic)
        w = min(p.n, (2 ** lev - 1) * (len(p.h) - 1) + 1)
        return w ** p.d

    def pick(lev, k):
        offs = levels[lev]
        out = []
        for _ in range(k):
            off, c = offs[int(rng.integers(len(offs)))]
            out.append(off + int(rng.integers(c)))
        return out

    per_unit, spent, sampled = {}, 0.0, 0
    for lev in lev_order:
        if lev > max(lev_order[0], lev_order[-1] - 2) and len(per_unit) >= 3:
            break                                   # the two coarsest levels: one unit costs ~1 min
        k = nthreads if lev == lev_order[0] or per_unit.get(lev - 1, 0) * nthreads < budget_s / 8 else 1
        units = pick(lev, k)
        t0 = time.perf_counter()
        rows = R.rows(p, units, nthreads=nthreads)
        for i, mu in enumerate(units):
            ret.retained_row(p, mu, rows[i])
        dt = time.perf_counter() - t0
        spent += dt
        sampled += len(units)
        per_unit[lev] = dt / max(len(units), nthreads)   # wall seconds per unit with every thread busy
    measured = sorted(per_unit)
    xs = np.array([supp(l) for l in measured], dtype=float)
    ys = np.array([per_unit[l] for l in measured])
    b, a = np.polyfit(xs, ys, 1) if len(measured) >= 2 else (0.0, ys[0])
    t_total_est = 0.0
    for lev in lev_order:
        t_unit = per_unit[lev] if lev in per_unit else a + b * supp(lev)
        t_total_est += t_unit * sum(c for _, c in levels[lev])
    extrap = [l for l in lev_order if l not in per_unit]
    nnz = p.N * p.band_L if p.retain == "band" else p.N * p.N
    return {"value": nnz / t_total_est, "unit": "entries/s", "cores": nthreads, "kind": "oracle",
            "sample": (f"{sampled} units over levels {measured} ({spent:.1f} s wall on {nthreads} threads); "
                       f"levels {extrap} extrapolated by t = a + b·|supp ψ| fitted on the measured levels; "
                       f"est. {t_total_est:.0f} s for all {p.N} units")}, t_total_est


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from synth import configs as C
    p = C.get(args.config)
    from oracle import rows as R
    R.build()
    cb, t_est = cpu_oracle_rate(p, budget_s=min(20.0, 4.0 * max(1, args.steps)))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "entries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_est * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, synth/configs.py)",
            "config": {"workload": WORKLOAD.get(args.config, args.config), "config": args.config},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2005_09870_b200 import Decomposition, Spec
    from synth import configs as C

    world, rank, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator set-up lines on stderr (evidence)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    p = C.get(args.config)
    u_d = torch.from_numpy(p.u).to(dev)
    v_d = torch.from_numpy(p.v).to(dev)
    spec = Spec(p.d, p.n, p.J, p.h, u_d, v_d, dtype=args.dtype, retain=p.retain, tau_rel=p.tau_rel,
                band_L=p.band_L, rank=rank, world=world, device=dev)
    dec = Decomposition(spec)
    dec.profile(True)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        dec.decompose(sp)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phase = np.zeros(3)
    lp_acc = []
    from paper_2005_09870_b200 import pcwd as PW
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with Clocks(dev) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))                    # L2 flush, outside the timed pair
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()                       # every rank starts the step together
            ev[i][0].record(stream)
            dec.decompose(sp)
            ev[i][1].record(stream)
            ev[i][1].synchronize()
            ms3, fma3 = dec.phase_times()
            phase += np.array(ms3)
            lp_acc.append(dec.launch_profile())
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = np.array([a.elapsed_time(b) for a, b in ev])
    info = dec.info()
    nnz = info.nnz
    launches = info.kernel_launches
    if world > 1:
        step_ms = PW.allreduce_max_vec(step_ms, dev)   # per step: the slowest rank (device time)
        offsets = PW.global_row_offsets(nnz, dev)     # C-b: all-gather of the per-rank nnz
        nnz_all = int(offsets[-1])
    else:
        offsets = [0, nnz]
        nnz_all = nnz
    t_ms = float(step_ms.sum())
    ms_per_step = t_ms / args.steps
    value = nnz_all / (ms_per_step * 1e-3)

    # dominant kernel: the unit-kernel launch with the largest time (CUDA events around each launch on the
    # decompose stream), FP32 FMA-pipe roofline; achieved = its algorithmic FMAs (SURVEY §8(d) per-unit
    # figure × its units) / its mean duration
    klist = [[0.0, 0.0, "", 0] for _ in lp_acc[0]] if lp_acc else []
    for lp in lp_acc:
        for i, (ms, fma, kind, lev) in enumerate(lp):
            klist[i][0] += ms / len(lp_acc)
            klist[i][1], klist[i][2], klist[i][3] = fma, kind, lev
    dom = max(klist, key=lambda x: x[1])   # the launch with the most algorithmic work (coarse levels may overlap)
    # per-kernel durations with the launches serialised (one extra, untimed decompose): the overlapped schedule's
    # per-launch events span the concurrent coarse streams, not the kernels' own times
    PW._check(PW.lib().pcwd_profile(dec._h, 2), "pcwd_profile")
    dec.decompose(sp)
    torch.cuda.synchronize(dev)
    serial = dec.launch_profile()
    PW._check(PW.lib().pcwd_profile(dec._h, 1), "pcwd_profile")
    alone_ms = next((m for (m, f, k, lv) in serial if (k, lv) == (dom[2], dom[3])), None)   # the dominant kernel alone
    ms_units = phase[1] / args.steps
    ms_tmpl = phase[0] / args.steps
    peaks = _peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12      # derived: SMs × lanes × 2 × clock
    if args.dtype == "f64":
        fp32_peak /= 2.0                                  # FP64 pipe: half the FP32 rate on B200 (ffma_peak: 36 TF)
    achieved = 2.0 * dom[1] / (dom[0] * 1e-3) / 1e12
    traffic, traffic_src = _ncu_traffic(dom[2], dom[3]) if args.dtype == "f32" else (None, None)
    roofline = {"bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": traffic,
                "traffic_source": f"{traffic_src} (dram__bytes_read.sum + dram__bytes_write.sum, one launch)"
                if traffic_src else None,
                "kernel": f"{dom[2]} unit kernel, level {dom[3]} (a2 k-sum + a3 cascade + a4 gather)",
                "kernel_ms": dom[0], "kernel_share_of_step": dom[0] / ms_per_step,
                "kernel_ms_alone": alone_ms, "frac_alone": (2.0 * dom[1] / (alone_ms * 1e-3) / 1e12 / fp32_peak
                                                            if alone_ms else None),
                "fma_per_launch": dom[1],
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 flop x sm_max_mhz of MEASURED_PEAKS.json"
                + (" / 2 (FP64)" if args.dtype == "f64" else ""),
                "all_unit_kernels": {"ms": ms_units, "tflops": 2.0 * fma3[1] / (ms_units * 1e-3) / 1e12,
                                     "frac": 2.0 * fma3[1] / (ms_units * 1e-3) / 1e12 / fp32_peak},
                "templates_ms": ms_tmpl,
                "launches": [{"kind": k, "level": lv, "ms": round(m, 4), "tflops": round(2 * f / (m * 1e-3) / 1e12, 2)}
                             for (m, f, k, lv) in serial],
                "launches_timing": "each unit-kernel launch alone (pcwd_profile(h, 2): serialised, CUDA events)",
                "hbm_achieved_gbs": info.bytes_algorithmic / (ms_per_step * 1e-3) / 1e9,
                "hbm_peak_gbs": peaks.get("hbm_gbs")}

    # e2e: through the public API with HOST buffers.  Per step: pcwd_set_kernels (H2D of this step's
    # u, v from pinned memory into the handle's plan) + pcwd_decompose_to_host (the CSR rows streamed to
    # pinned host buffers as each launch finishes); the plan (handle) is built once, as a user
    # decomposing a sequence of operators of one geometry does.  `with_create_ms`: the same step with
    # pcwd_create (host planning + allocation) inside the timed region, and the unoverlapped copy.
    e2e = None
    if not args.no_e2e:
        u_h = torch.from_numpy(p.u).pin_memory()
        v_h = torch.from_numpy(p.v).pin_memory()
        meta = dec.csr_meta()
        rp_h = torch.empty(meta.n_rows + 1, dtype=torch.int64).pin_memory()
        col_h = torch.empty(meta.nnz, dtype=torch.int32).pin_memory()
        val_h = torch.empty(meta.nnz, dtype=torch.float32 if args.dtype == "f32" else torch.float64).pin_memory()
        from paper_2005_09870_b200 import pcwd as P
        import ctypes

        def spec_h():
            return Spec(p.d, p.n, p.J, p.h, u_h.numpy(), v_h.numpy(), dtype=args.dtype, retain=p.retain,
                        tau_rel=p.tau_rel, band_L=p.band_L, rank=rank, world=world, device=dev)
        dplan = Decomposition(spec_h())
        # u_k as the compact impulse responses they are: each step's u is handed over on the plan's
        # periodic bounding box (pcwd_set_kernels_box), built once here as the caller's own storage of u
        (lo0, lo1), (w0, w1) = dplan.kernel_box()
        ufull = p.u.reshape(p.u.shape[0], p.n, p.n) if p.d == 2 else p.u.reshape(p.u.shape[0], 1, p.n)
        ubox_h = torch.from_numpy(np.ascontiguousarray(
            ufull[:, (lo0 + np.arange(w0)) % ufull.shape[1]][:, :, (lo1 + np.arange(w1)) % p.n])).pin_memory()
        times = []
        for i in range(max(3, min(args.steps, 10)) + 1):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            dplan.set_kernels(u_h, v_h, sp)
            dplan.decompose_to_host(rp_h, col_h, val_h, sp)
            torch.cuda.synchronize(dev)
            times.append(time.perf_counter() - t0)
        # BAND / FULL: the retained pattern (row_ptr, col) is index-defined — a function of the plan alone — so a
        # sequence of operators on one plan needs it once; the per-step result is then the values (NULL row_ptr /
        # col skip those arrays in pcwd_decompose_to_host)
        fixed_pattern = p.retain in ("band", "full")
        times_v = []
        if fixed_pattern:
            for i in range(max(3, min(args.steps, 10)) + 1):
                torch.cuda.synchronize(dev)
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                dplan.set_kernels_box(ubox_h, v_h, sp)
                dplan.decompose_to_host(None, None, val_h, sp)
                torch.cuda.synchronize(dev)
                times_v.append(time.perf_counter() - t0)
        dplan.close()
        times = np.array(times[1:])
        if world > 1:
            times = PW.allreduce_max_vec(times, dev)     # per step: the slowest rank's copy-in + decompose + copy-out
        t_full = float(np.median(times))
        t_e2e = t_full
        if fixed_pattern:
            times_v = np.array(times_v[1:])
            if world > 1:
                times_v = PW.allreduce_max_vec(times_v, dev)
            t_e2e = float(np.median(times_v))
        times_c = []
        for i in range(3):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            d2 = Decomposition(spec_h())
            d2.decompose(sp)
            P._check(P.lib().pcwd_copy_csr(d2._h, rp_h.data_ptr(), col_h.data_ptr(), val_h.data_ptr(),
                                           ctypes.c_void_p(sp)), "copy")
            torch.cuda.synchronize(dev)
            times_c.append(time.perf_counter() - t0)
            d2.close()
        times_c = np.array(times_c[1:])
        if world > 1:
            times_c = PW.allreduce_max_vec(times_c, dev)
        h2d_full = int(p.u.nbytes + p.v.nbytes) * world
        h2d = int(ubox_h.numel() * 8 + p.v.nbytes) * world if fixed_pattern else h2d_full
        d2h_full = int(rp_h.numel() * 8 + col_h.numel() * 4 + val_h.numel() * val_h.element_size())
        d2h = int(val_h.numel() * val_h.element_size()) if fixed_pattern else d2h_full
        if world > 1:
            d2h = int(PW.allreduce_sum(float(d2h), dev))
            d2h_full = int(PW.allreduce_sum(float(d2h_full), dev))
        e2e = {"value": nnz_all / t_e2e, "unit": "entries/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": t_e2e * 1e3,
               "calls": ("pcwd_set_kernels_box (u_k on the plan's support box) + pcwd_decompose_to_host (plan built "
                         "once); the index-defined band pattern (row_ptr, col) is copied once per plan, the values "
                         "every step") if fixed_pattern else
                        "pcwd_set_kernels + pcwd_decompose_to_host (plan built once)",
               "full_csr_every_step": {"value": nnz_all / t_full, "ms_per_step": t_full * 1e3,
                                       "calls": "pcwd_set_kernels (whole u) + pcwd_decompose_to_host (full CSR)",
                                       "h2d_bytes_per_step": h2d_full, "d2h_bytes_per_step": d2h_full},
               "with_create_ms": float(np.median(times_c)) * 1e3,
               "timing": "wall clock per rank, synchronize on both sides, max over ranks per step, median"}

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu:
            cb, _ = cpu_oracle_rate(p, budget_s=15.0)
        line = {"metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (seeded, synth/configs.py; no dataset in the paper's path)",
                "config": {"workload": WORKLOAD.get(args.config, args.config), "config": args.config,
                           "units": p.N, "retained_per_unit": p.band_L, "nnz": nnz_all,
                           "l2": "flushed (256 MiB write) before every timed step",
                           "sharding": f"{world} rank(s), cost-balanced contiguous unit ranges",
                           "row_offsets": [int(x) for x in offsets]},
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": launches * args.steps, "clocks": clk.summary(),
                "decomposition_time_s": ms_per_step * 1e-3}
        print(json.dumps(line), flush=True)
    dec.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"], help="compute dtype (the headline is f32)")
    args = ap.parse_args()
    rc = relaunch_under_torchrun(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
