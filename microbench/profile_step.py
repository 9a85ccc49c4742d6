"""One hot-path step (iga_assemble + iga_sensitivity) on a config, for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:k3_contract -c 1 \
        -o gpurun_out/x python microbench/profile_step.py --config 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--no-sensitivity", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2107_09568_b200 import Assembler
    from synth import make_config, draw_uv_seeded
    prob = make_config(args.config)
    A = Assembler(prob)
    s = A.sizes
    dev = torch.device("cuda")
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    u, v = draw_uv_seeded(args.config, s.n_dof)
    u, v = torch.tensor(u, device=dev), torch.tensor(v, device=dev)
    grad = torch.empty(s.n_macro_cp * prob.d, dtype=torch.float64, device=dev)
    for _ in range(args.reps):
        A.assemble(ctrl, young, prob.nu, vals)
        if not args.no_sensitivity:
            A.sensitivity(ctrl, young, prob.nu, u, v, grad)
    torch.cuda.synchronize()
    print("sizes: tiles", s.n_tiles, "rows", s.n_local_rows, "nnz", s.nnz, "multi blocks", s.n_multi_blocks,
          "side slots", s.n_side_slots, "contrib", s.n_contrib)


if __name__ == "__main__":
    main()
