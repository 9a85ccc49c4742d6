"""Per-kernel device times (libiga's CUDA events) of iga_assemble + iga_sensitivity on a config."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--apply", action="store_true")
    ap.add_argument("--local", action="store_true", help="also time the nzdata-only assemble (K2 + K3 EPI 0)")
    ap.add_argument("--q", type=int, default=None, help="projection degree override (e.g. the Eq. 65 choice)")
    args = ap.parse_args()
    import torch
    from paper_2107_09568_b200 import Assembler
    from synth import make_config, draw_uv_seeded
    prob = make_config(args.config, q=args.q)
    A = Assembler(prob)
    s = A.sizes
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    u, v = draw_uv_seeded(args.config, s.n_dof)
    u, v = torch.tensor(u, device=dev), torch.tensor(v, device=dev)
    grad = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device=dev)
    y = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * prob.d ** 2, dtype=torch.float64, device=dev) if args.local else None
    for it in range(2):
        A.set_profiling(it == 1)
        for _ in range(args.reps if it else 2):
            A.assemble(ctrl, young, prob.nu, vals)
            A.sensitivity(ctrl, young, prob.nu, u, v, grad)
            if args.apply:
                A.apply(ctrl, young, prob.nu, u, y)
            if args.local:
                A.assemble(ctrl, young, prob.nu, None, local)
        torch.cuda.synchronize()
    ms, n = A.kernel_times()
    names = ["K2", "K3", "K4", "K5a", "K5b", "K5c", "stage", "K5x", "K3local", "apply"]
    flops = 2.0 * s.n_local_rows * s.n_k * s.n_tiles * prob.d ** 2
    out = {nm: round(ms[i] / max(n[i], 1), 4) for i, nm in enumerate(names) if n[i]}
    out["K3_tflops"] = round(flops / (out["K3"] * 1e-3) / 1e12, 2)
    out["K5a_tflops"] = round(flops / (out["K5a"] * 1e-3) / 1e12, 2)
    print(os.environ.get("IGA_LIB", "libiga.so"), json.dumps(out))


if __name__ == "__main__":
    main()
