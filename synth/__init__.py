"""Seeded synthetic inputs (placement and random draws only; no method arithmetic)."""
from .configs import (Problem, Spline, Interface, make_config, draw_uv, draw_uv_seeded,  # noqa: F401
                      open_uniform_knots, greville)
