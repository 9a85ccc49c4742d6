"""E_proj (Eq. 59) and the Eq. 65 degree selection for the bench configs, on the GPU
(iga_projection_error / iga_select_degree); prints one JSON line per config."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2107_09568_b200 import projection_error, select_degree
from synth import make_config

for c in (1, 2, 3, 4, 5):
    prob = make_config(c)
    q = prob.q
    projection_error(prob.macro, q, prob.nu, n_samples=8)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = projection_error(prob.macro, q, prob.nu, n_samples=8)
    dt = time.perf_counter() - t0
    sel = {}
    for tol in (1e-2, 1e-3, 1e-4):
        try:
            qs, es = select_degree(prob.macro, prob.nu, tol, n_samples=8)
            sel[str(tol)] = {"q": list(qs), "E_proj": es}
        except Exception as ex:   # tolerance not reachable below q = 4
            sel[str(tol)] = {"error": str(ex)[:80]}
    print(json.dumps({"config": c, "n_tiles": prob.n_tiles, "q": q, "E_proj": e, "ms": dt * 1e3,
                      "select": sel}), flush=True)
