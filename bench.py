"""bench.py — K formation (+ sensitivity) throughput of libiga on B200.

Workload (default): BASELINE.json configs[4] = cfg5 — cfg3's quarter-annulus macro map
refined to 32×16×16 elements (8192 tiles) with the 6-strut lattice tile, p = q = 2,
FP64, plus uᵀ(∂K/∂P)v with seeded N(0,1) u, v.  One step = the whole hot path of
SURVEY.md §8(a) rows a2-a5: K2 interpolation -> K3 DMMA contraction -> K4 CSR gather
(iga_assemble) and K5a -> K5b -> K5c (iga_sensitivity).  Row a1 (tables) is offline per
the paper and reported separately (`offline`).

Timing: W warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA
events on the launching stream, max over ranks.  The working set (CSR values 22.9 GB,
X 12 GB) is >> the 126 MB L2, so no explicit flush is needed.
Per-kernel device times come from libiga's own CUDA events on the same stream
(iga_set_profiling) over the timed region.

--impl reference: the oracle (oracle/, NumPy FP64) on host cores, on a bounded sample
of the same workload (cfg5 generator at a reduced macro grid), same metric/unit.
Multi-GPU (torchrun): every rank forms K and g for its own problem instance (weak
scaling, no data-path collective); value = all ranks' tiles / max-over-ranks time.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.15      # measured DMMA ceiling, profiles/r01_fp64_ceiling.md
METRIC = "K formation tiles/s and nnz/s at 1 B200; % of FP64-tensor / HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-sensitivity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--select-degree", type=float, default=None, metavar="TOL",
                    help="choose the projection degree per direction a priori (Eq. 65, iga_select_degree) "
                         "for E_proj <= TOL instead of the config's q (not the BASELINE configuration)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: shard ONE problem over the ranks (slabs + halo, gradient all-reduce; "
                         "strong scaling) instead of one independent problem per rank (weak scaling)")
    return ap.parse_args()


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend)
    return rank, world


def reduce_max(x, world):
    """Max over ranks of a float (device timing rule)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x, world):
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def algorithmic(prob, s, sens):
    """Algorithmic work per launch.  The contraction is
    the Eq. 38-reduced one: per table row and tile, n_π·(n_p1² + n_p2²) multiply-adds (45 n_π
    in 3D: the distinct components of Ā, Eq. 38) instead of Eq. 58's d² n_π · d² = 81 n_π;
    `eq58_flops` is the unreduced count of SURVEY §8(d), reported for reference only."""
    d = prob.d
    dd = d * d
    N = s.n_tiles * dd
    n_pi = s.n_k // dd
    n_sym = (d * (d + 1) // 2) ** 2 + (d * (d - 1) // 2) ** 2          # 45 (3D), 10 (2D)
    gemm = 2.0 * s.n_local_rows * s.n_tiles * n_sym * n_pi            # reduced, unpadded
    eq58 = 2.0 * s.n_local_rows * s.n_k * N
    k2_bytes = 8.0 * (s.n_tiles * n_sym * n_pi + s.n_tiles + s.n_macro_cp * d)
    # K3 epilogue: CSR writes of the single-contribution blocks, side-slot writes, rank map
    multi_vals = 2.0 * s.n_multi_blocks * dd                      # (I,J) and (J,I) (diag: once, ignored)
    k3_bytes = 8.0 * (s.nnz - multi_vals) + 8.0 * dd * s.n_side_slots + 4.0 * s.n_local_rows * s.n_tiles
    # K4: side-slot reads + the multi blocks' CSR writes + their descriptors
    k4_bytes = 8.0 * dd * s.n_side_slots + 8.0 * multi_vals + 28.0 * s.n_multi_blocks + 1.0 * s.n_side_slots
    # K5x: X writes (rows x tiles x d²) + u, v reads
    k5x_bytes = 8.0 * s.n_local_rows * N + 16.0 * s.n_dof
    return dict(k3_flops=gemm, k5a_flops=gemm if sens else 0.0, k2_bytes=k2_bytes, k3_bytes=k3_bytes,
                k4_bytes=k4_bytes, k5x_bytes=k5x_bytes if sens else 0.0, eq58_flops=eq58)


def load_traffic():
    """dram bytes per launch from the committed ncu --set full summary (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def _oracle_sample(n_el):
    from oracle import assemble as As
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config, draw_uv_seeded
    prob = make_config(5, n_el=n_el)
    dm = DofMap(prob)
    tabs = As.Tables(prob)
    pt = Pattern(prob, dm, tabs.pairs)
    u, v = draw_uv_seeded(5, dm.n_dof)
    return prob, tabs, pt, u, v


def cpu_baseline_oracle(n_el=(8, 4, 4), sens=True, parallel=False):
    """The oracle (NumPy FP64, as it stands) on a bounded sample of the cfg5 workload:
    the cfg5 generator (same tile, p=q=2) at a reduced macro grid.  Tables, DofMap and
    pattern are built untimed (offline, as for the GPU).  Timed: K^π (interpolation,
    table·coefficient product, CSR scatter) + g = uᵀ(∂K^π/∂P)v for every coordinate.
    parallel=False: one host thread (BLAS limited to 1 thread; the paper's serial setting,
    P:459).  parallel=True: the same oracle calls over tiles (element matrices, gradient
    terms) and node ranges (scatter) in a fork pool of one single-threaded process per
    host core (tests/parity_tools.py).  Returns (tiles, seconds, cores, nnz)."""
    from threadpoolctl import threadpool_limits
    from oracle import assemble as As, sensitivity as S
    prob, tabs, pt, u, v = _oracle_sample(n_el)
    if not parallel:
        with threadpool_limits(1):
            t0 = time.perf_counter()
            As.assemble_lookup(prob, tabs, pt)
            if sens:
                S.sensitivity(prob, tabs, pt, u, v)
            dt = time.perf_counter() - t0
        return prob.n_tiles, dt, 1, pt.nnz
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import parity_tools as PT
    d = prob.d
    t0 = time.perf_counter()
    local = PT.shared_array((prob.n_tiles, pt.n_rows_tile, d, d), np.float64)
    PT.run(PT.w_local, PT.tile_chunks(prob.n_tiles, 2), prob=prob, tabs=tabs, local=local)
    bm = PT.shared_array((prob.n_tiles * pt.n_rows_tile, 2), np.int64)     # (offline on the GPU side)
    PT.run(PT.w_block_map, PT.tile_chunks(prob.n_tiles, 8), pattern=pt, bm=bm)
    t_bm = time.perf_counter()
    vals = PT.shared_array((pt.nnz,), np.float64)
    PT.run(PT.w_scatter, PT.node_ranges(pt, d, PT.n_workers()), prob=prob, pattern=pt, local=local, bm=bm, vals=vals)
    t1 = time.perf_counter()
    if sens:
        np.sum(PT.run(PT.w_sensitivity, PT.tile_chunks(prob.n_tiles, 2), prob=prob, tabs=tabs, pattern=pt, u=u, v=v),
               axis=0)
    dt = time.perf_counter() - t1 + (t_bm - t0)
    return prob.n_tiles, dt, PT.n_workers(), pt.nnz


def oracle_t_cost(n_std_tiles=4):
    """On-box T_cost (Eq. 64) of the oracle: time per tile of the standard full-Gauss
    element matrices K^• (same n_g as the tables) over the lookup K^π (interpolation,
    table product and scatter), both the plain NumPy oracle on the host cores, on the cfg5
    tile.  K^• is timed on n_std_tiles tiles and the lookup on the 8-tile sample (per-tile
    cost is uniform); quoted beside the paper's 11-107x (serial laptop CPU)."""
    from oracle import assemble as As
    from oracle.dofmap import DofMap, Pattern
    from synth import make_config
    prob = make_config(5, n_el=(2, 2, 2))
    tabs = As.Tables(prob)
    pt = Pattern(prob, DofMap(prob), tabs.pairs)
    t0 = time.perf_counter()
    As.assemble_lookup(prob, tabs, pt)
    t_pi = (time.perf_counter() - t0) / prob.n_tiles
    pts = As._tile_points(prob, prob.n_gauss)
    t0 = time.perf_counter()
    for t in range(n_std_tiles):
        As.local_standard(prob, t, tabs.pairs, pts=pts)
    t_std = (time.perf_counter() - t0) / n_std_tiles
    return {"t_cost": t_std / t_pi, "s_per_tile_standard": t_std, "s_per_tile_lookup": t_pi,
            "tiles_timed": {"standard": n_std_tiles, "lookup": prob.n_tiles},
            "note": "oracle K^bullet / oracle K^pi per tile on the host (Eq. 64), K^bullet timed on a subset of "
                    "tiles (per-tile cost is uniform); paper: 11-107x serial"}


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    n_el = (8, 4, 4)
    times = []
    n_tiles = nnz = cores = None
    for i in range(args.warmup + args.steps):
        n_tiles, dt, cores, nnz = cpu_baseline_oracle(n_el=n_el, sens=not args.no_sensitivity, parallel=True)
        if i >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    value = n_tiles / t
    sample = (f"cfg5 generator at macro grid {n_el} ({n_tiles} tiles, nnz {nnz}): oracle K^pi "
              f"(interpolation + table product + CSR scatter)" + ("" if args.no_sensitivity else " + full gradient")
              + f"; tables/DofMap/pattern untimed (offline); tiles and node ranges over a pool of {cores} "
              "single-threaded host processes")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tiles/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg5-sample{n_el}", "n_tiles": n_tiles, "nnz": nnz, "p": 2, "q": 2},
            "nnz_per_s": nnz / t,
            "cpu_baseline": {"value": value, "unit": "tiles/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tiles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import torch
    from paper_2107_09568_b200 import Assembler
    from synth import make_config, draw_uv_seeded

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sens = not args.no_sensitivity
    prob = make_config(args.config)
    q_sel = None
    if args.select_degree is not None:   # Eq. 65 a-priori degree (device E_proj, untimed like the tables)
        from paper_2107_09568_b200 import select_degree
        q_sel, e_sel = select_degree(prob.macro, prob.nu, args.select_degree)
        prob = make_config(args.config, q=q_sel if len(set(q_sel)) > 1 else q_sel[0])
    shard = args.shard and world > 1
    t0 = time.perf_counter()
    A = Assembler(prob, shard=(world, rank) if shard else None)
    build_s = time.perf_counter() - t0
    s = A.sizes
    if shard:
        from paper_2107_09568_b200.shard import allreduce_grad
    d = prob.d
    ctrl = torch.tensor(prob.macro.ctrl, dtype=torch.float64, device=dev)
    young = torch.tensor(prob.young, dtype=torch.float64, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    u_np, v_np = draw_uv_seeded(args.config, s.n_dof)
    u = torch.tensor(u_np, device=dev)
    v = torch.tensor(v_np, device=dev)
    grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        if sens:   # K and g in one call (iga_assemble_sensitivity)
            A.assemble_sensitivity(ctrl, young, prob.nu, u, v, vals, grad, stream=stream)
            if shard:
                allreduce_grad(grad, world)   # the sharded step's one collective (NCCL)
        else:
            A.assemble(ctrl, young, prob.nu, vals, stream=stream)

    def timed_loop(fn, steps):
        """steps calls of fn on `stream`, an event before each and one after the last:
        (total ms / steps, per-step ms list), barrier + synchronize on both sides."""
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        barrier(world)
        torch.cuda.synchronize()
        for i in range(steps):
            evs[i].record(stream)
            fn()
        evs[steps].record(stream)
        torch.cuda.synchronize()
        barrier(world)
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
        return evs[0].elapsed_time(evs[steps]) / steps, per

    def window(per, mean, n_tiles_w, nnz_w):
        med, best = float(np.median(per)), float(np.min(per))
        med_g, best_g, mean_g = reduce_max(med, world), reduce_max(best, world), reduce_max(mean, world)
        return {"ms_mean": mean_g, "ms_median": med_g, "ms_best": best_g,
                "tiles_per_s_median": n_tiles_w / (med_g * 1e-3), "tiles_per_s_best": n_tiles_w / (best_g * 1e-3),
                "nnz_per_s_median": nnz_w / (med_g * 1e-3) if nnz_w else None, "steps": len(per)}

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    A.set_profiling(True)
    clocks = ClockSampler(local_rank)
    ms_local, per_main = timed_loop(step, args.steps)    # THE timed region: K steps of the whole hot path
    clk = clocks.stop()
    kms, kn = A.kernel_times()
    A.set_profiling(False)
    ms = reduce_max(ms_local, world)
    tiles_total = s.n_tiles if shard else s.n_tiles * world   # shard: the ranks share one problem
    nnz_total = reduce_sum(s.nnz, world) if shard else s.nnz * world
    value = tiles_total / (ms * 1e-3)
    nnz_per_s = nnz_total / (ms * 1e-3)

    # ---- SURVEY §8(d) windows, each its own CUDA-event loop (median and best) --------
    windows = {("K_plus_g" if sens else "K_formation"): window(per_main, ms_local, tiles_total, nnz_total)}
    if sens:
        for _ in range(2):
            A.assemble(ctrl, young, prob.nu, vals, stream=stream)
        m, per = timed_loop(lambda: A.assemble(ctrl, young, prob.nu, vals, stream=stream), args.steps)
        windows["K_formation"] = window(per, m, tiles_total, nnz_total)
    if not shard:
        try:
            local_buf = torch.empty(s.n_local_rows * s.n_tiles_local * d * d, dtype=torch.float64, device=dev)
        except RuntimeError:
            local_buf = None
        if local_buf is not None:
            nz = lambda: A.assemble(ctrl, young, prob.nu, None, local_buf, stream=stream)
            for _ in range(2):
                nz()
            m, per = timed_loop(nz, args.steps)
            windows["non_zeros"] = window(per, m, tiles_total, None)
            windows["non_zeros"]["local_values"] = int(s.n_local_rows * s.n_tiles_local * d * d) * world
            del local_buf
            torch.cuda.empty_cache()
    if not shard:   # the matrix-free product y = K u (Eq. 74), K never stored
        y_buf = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
        mf = lambda: A.apply(ctrl, young, prob.nu, u, y_buf, stream=stream)
        for _ in range(2):
            mf()
        m, per = timed_loop(mf, args.steps)
        windows["matrix_free_apply"] = window(per, m, tiles_total, None)
        del y_buf
    windows["note"] = ("non_zeros = K2 + K3 into the element matrices, no CSR (the paper's convention, P:457); "
                       "K_formation = K2 + K3 + K4 into CSR (iga_assemble, the metric's name); K_plus_g = the "
                       "bench step (iga_assemble_sensitivity, BASELINE cfg5: K and the gradient) whose mean is `value`; "
                       "matrix_free_apply = one y = K u without forming K (iga_apply, Eq. 74)")

    # ---- e2e: host (pinned) inputs through the C ABI, gradient read back ---------
    e2e = None
    if not args.no_e2e:
        h_ctrl = torch.tensor(prob.macro.ctrl, dtype=torch.float64).pin_memory()
        h_young = torch.tensor(prob.young, dtype=torch.float64).pin_memory()
        h_u = torch.tensor(u_np).pin_memory()
        h_v = torch.tensor(v_np).pin_memory()
        h_grad = torch.empty(s.n_macro_cp * d, dtype=torch.float64).pin_memory()
        h_grad_np = h_grad.numpy()

        def step_e2e():
            if sens:
                A.assemble_sensitivity(h_ctrl.numpy(), h_young.numpy(), prob.nu, h_u.numpy(), h_v.numpy(), vals,
                                       h_grad_np, stream=stream)
                if shard:
                    gd = torch.from_numpy(h_grad_np).to(dev)
                    allreduce_grad(gd, world)
                    h_grad.copy_(gd)
            else:
                A.assemble(h_ctrl.numpy(), h_young.numpy(), prob.nu, vals, stream=stream)
        step_e2e()
        m, _ = timed_loop(step_e2e, args.steps)
        ms_e2e = reduce_max(m, world)
        # staged by the library once per call: P (n_cp·d), E (n_tiles), u and v (n_dof each)
        h2d = 8 * (s.n_macro_cp * d + s.n_tiles + (2 * s.n_dof if sens else 0))
        e2e = {"value": tiles_total / (ms_e2e * 1e-3), "unit": "tiles/s", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * s.n_macro_cp * d if sens else 0),
               "note": "inputs P, E (and u, v) from pinned host memory via the C ABI [any]-pointer staging; "
                       "K stays device-resident (consumer is a GPU solver / matrix-free); gradient read back"}

    alg = algorithmic(prob, s, sens)
    per = lambda slot: kms[slot] / max(kn[slot], 1)
    k3_ms, k5a_ms, k2_ms, k4_ms, k5x_ms = per(1), per(3), per(0), per(2), per(7)
    traffic = load_traffic()
    rooflines = {
        "K3_contraction_scatter": {"bound": "tensor", "achieved": alg["k3_flops"] / (k3_ms * 1e-3) / 1e12,
                                   "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "ms": k3_ms,
                                   "epilogue_hbm_gbs": alg["k3_bytes"] / (k3_ms * 1e-3) / 1e9},
        "K2_interpolation": {"bound": "hbm", "achieved": alg["k2_bytes"] / (k2_ms * 1e-3) / 1e9,
                             "peak": None, "unit": "GB/s", "ms": k2_ms},
        "K4_multi_gather": {"bound": "hbm", "achieved": alg["k4_bytes"] / (k4_ms * 1e-3) / 1e9,
                            "peak": None, "unit": "GB/s", "ms": k4_ms},
    }
    if sens:
        fused = kn[7] == 0   # K5g: X̃ generated in shared memory inside the sensitivity GEMM
        if not fused:
            rooflines["K5x_generate_X"] = {"bound": "hbm", "achieved": alg["k5x_bytes"] / (k5x_ms * 1e-3) / 1e9,
                                           "peak": None, "unit": "GB/s", "ms": k5x_ms}
        rooflines["K5g_X_and_W_gemm" if fused else "K5a_W_gemm"] = {
            "bound": "tensor", "achieved": alg["k5a_flops"] / (k5a_ms * 1e-3) / 1e12,
            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "ms": k5a_ms,
            **({"note": "K5x fused: the X-tilde generator warps share the FP64 pipe with the DMMAs"} if fused else {})}
        rooflines["K5b_reverse"] = {"ms": per(4)}
        rooflines["K5c_reduce"] = {"ms": per(5)}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = peaks.get("hbm_gbs")
    except Exception:
        hbm = None
    hbm_source = "MEASURED_PEAKS.json hbm_gbs" if hbm else "of fallback (B200_PROFILING.md: 6.65 TB/s; MEASURED_PEAKS.json absent)"
    hbm = hbm or 6650.0
    for k in ("K2_interpolation", "K4_multi_gather", "K5x_generate_X"):
        if k in rooflines:
            rooflines[k]["peak"] = hbm
    for k, r in rooflines.items():
        if r.get("peak"):
            r["frac"] = r["achieved"] / r["peak"]
            # SURVEY §8(d)'s second denominators: the datasheet FP64 tensor 40 TF/s, BASELINE's 8 TB/s
            if r["unit"] == "TFLOP/s":
                r["frac_vs_datasheet_40tf"] = r["achieved"] / 40.0
            else:
                r["frac_vs_8tbs"] = r["achieved"] / 8000.0
    dom = rooflines["K3_contraction_scatter"]
    # K3's bound: the roof whose time is larger (tensor at the BASELINE q = 2; at q = 1, the
    # Eq. 65 choice for cfg5, its 23 GB CSR epilogue takes longer than its flops)
    k3_hbm_bound = alg["k3_bytes"] / (hbm * 1e9) > alg["k3_flops"] / (FP64_PEAK_TFLOPS * 1e12)
    if k3_hbm_bound:
        dom = dict(dom, bound="hbm", achieved=alg["k3_bytes"] / (k3_ms * 1e-3) / 1e9, peak=hbm, unit="GB/s")
        dom["frac"] = dom["achieved"] / hbm
        rooflines["K3_contraction_scatter"]["bound_note"] = "HBM-bound at this q: the CSR epilogue bytes take longer than the flops"
    roofline = {"bound": dom["bound"], "kernel": "K3 contraction (FP64 DMMA) + fused CSR scatter", "achieved": dom["achieved"],
                "peak": dom["peak"], "unit": dom["unit"], "frac": dom["frac"],
                # the committed ncu capture is of the default (BASELINE) configuration only
                "traffic": traffic.get("K3_dram_bytes_per_launch") if q_sel is None and args.config == 5 else None,
                "peak_source": (hbm_source if k3_hbm_bound else
                                "measured DMMA ceiling, profiles/r01_fp64_ceiling.md (MEASURED_PEAKS.json has no FP64 entry)"),
                "algorithmic_flops_per_launch": alg["k3_flops"], "algorithmic_bytes_per_launch": alg["k3_bytes"],
                "flops_note": "Eq. 38-reduced contraction (45 n_pi MACs per table row and tile in 3D); "
                              "the unreduced Eq. 58 product would be %.4g flop, i.e. %.2f TFLOP/s equivalent"
                              % (alg["eq58_flops"], alg["eq58_flops"] / (k3_ms * 1e-3) / 1e12)}

    line = {"metric": METRIC, "value": value, "unit": "tiles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg{args.config}" + ("" if sens else " (K only)")
                       + (f" with the Eq. 65 degree q={list(q_sel)} (tol {args.select_degree:g}, E_proj {e_sel:.2e})"
                          if q_sel is not None else ""),
                       "parallelism": (f"slab{world} (one problem: slabs + halo, gradient all-reduce)" if shard
                                       else f"replica{world} (one independent problem per GPU)"),
                       "n_tiles_per_gpu": int(s.n_tiles_owned if shard else s.n_tiles), "nnz": int(nnz_total),
                       "n_dof": int(s.n_dof), "p": prob.p,
                       "q": prob.q, "sensitivity": sens,
                       "l2": "working set >> 126 MB L2 (CSR values alone 8*nnz bytes); no explicit flush"},
            "nnz_per_s": nnz_per_s, "windows": windows, "roofline": roofline, "rooflines_all": rooflines,
            "clocks": clk, "e2e": e2e,
            "gpu_launches": int(sum(kn[i] for i in (0, 1, 2, 3, 4, 5, 7))),   # libiga kernels in the timed region
            "kernel_ms_per_step": {"K2": k2_ms, "K3": k3_ms, "K4": k4_ms, "K5x (0: fused into K5g)": k5x_ms if sens else 0.0,
                                   "K5a": k5a_ms if sens else 0.0, "K5b": per(4) if sens else 0.0,
                                   "K5c": per(5) if sens else 0.0},
            "offline": {"build_s (host topology + K1 tables + pattern)": build_s}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_t, dt1, _, nnz = cpu_baseline_oracle(sens=sens)
        n_t, dtp, cores, _ = cpu_baseline_oracle(sens=sens, parallel=True)
        what = "oracle K^pi" + (" + full gradient" if sens else "")
        line["cpu_baseline"] = {
            "value": n_t / dtp, "unit": "tiles/s", "cores": cores, "kind": "oracle",
            "sample": f"cfg5 generator at macro grid (8,4,4) = {n_t} tiles (nnz {nnz}), {what}: {dtp:.2f} s over a "
                      f"fork pool of {cores} single-threaded processes (tiles / node ranges); tables/pattern untimed",
            "single_thread": {"value": n_t / dt1, "unit": "tiles/s", "cores": 1, "seconds": dt1,
                              "note": "same sample, one host thread (BLAS limited to 1), the paper's serial setting (P:459)"},
            "extrapolated_cfg5_s": {"single_thread": 8192 * dt1 / n_t, "all_cores": 8192 * dtp / n_t,
                                    "extrapolated": True,
                                    "note": "linear extrapolation to the 8192 cfg5 tiles (per-tile cost is uniform); "
                                            "the full cfg5 oracle is not run here"},
            "oracle_t_cost": oracle_t_cost()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
