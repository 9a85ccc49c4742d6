"""A small end-to-end run of every entry point (for compute-sanitizer memcheck/racecheck):
cfg1 and a small cfg2/cfg3/aniso problem through assemble (+nzdata), sensitivity, the one-call
step, apply, volume, load vector, L2 projection, E_proj and degree selection."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2107_09568_b200 import Assembler, projection_error, select_degree
from synth import make_config, draw_uv_seeded

dev = torch.device("cuda")
for c, kw, m in [(1, {}, 0), (2, dict(n_el=(2, 2, 1)), 0), (3, dict(n_el=(2, 1, 1)), 0),
                 (2, dict(n_el=(2, 1, 1), q=(1, 2, 3)), 0), (2, dict(n_el=(2, 1, 1)), 4)]:
    prob = make_config(c, **kw)
    A = Assembler(prob)
    if m:
        A.set_projection(m)
    s = A.sizes
    d = prob.d
    ctrl = torch.tensor(prob.macro.ctrl, device=dev)
    young = torch.tensor(prob.young, device=dev)
    vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
    local = torch.empty(s.n_local_rows * s.n_tiles * d * d, dtype=torch.float64, device=dev)
    A.assemble(ctrl, young, prob.nu, vals, local)
    u, v = draw_uv_seeded(c, s.n_dof)
    u, v = torch.tensor(u, device=dev), torch.tensor(v, device=dev)
    g = torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev)
    A.sensitivity(ctrl, young, prob.nu, u, v, g)
    A.assemble_sensitivity(ctrl, young, prob.nu, u, v, vals, g)
    y = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
    A.apply(ctrl, young, prob.nu, u, y)
    A.volume(ctrl, torch.empty(s.n_macro_cp * d, dtype=torch.float64, device=dev))
    f = torch.empty(s.n_dof, dtype=torch.float64, device=dev)
    A.load_vector(ctrl, [0.0, -1.0, 0.0][:d], f)
    coef = torch.zeros(s.n_tiles * d * d * s.k_stride, dtype=torch.float64, device=dev)
    A.interpolate(ctrl, young, prob.nu, coef)
    torch.cuda.synchronize()
    print("ok", c, kw, m, float(vals.abs().sum()), float(g.abs().sum()), flush=True)
prob = make_config(1)
print("E_proj", projection_error(prob.macro, (3, 1), prob.nu, n_samples=5), select_degree(prob.macro, prob.nu, 1e-3, n_samples=5))
