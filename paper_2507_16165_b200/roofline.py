"""Algorithmic FP64 flop accounting for the roofline.

Counts are per the normative operation order of the kernels (= the oracle):
an fma is 2 flops, every other +,-,*,/,sqrt is 1; transcendentals
(sin/cos/atan2/asin/pow), comparisons, fabs/fmin/fmax and integer work are 0.
Loop invariants (3M, h/2, h/6) are counted once per ray, i.e. not per step.

per step attempt (accepted or rejected):
  RKF45     137  = 6 rhs x 3 + stage sums 70 + 5th-order 22 + error 20
                   + scales 4 + guard 1 + h update 1 + phi update 1
  RK4        39  = 4 rhs x 3 + stage inputs 12 + combination 14 + phi 1
  REFERENCE 152  = DOPRI5 step incl. error norm and PI control
per ray (counted from the kernels' normative operation order, round 2):
  scene modes (RK4 / RKF45) 79 = raw camera direction 30 (u, v with the
    reciprocal correction, the three-vector sum) + orbital frame 29
    (scene_frame: dots, |T|^2, |D|^2 test, sqrt, one reciprocal, e2, u0')
    + plane normal 9 + first integral 8 + disk-line norm test 3;
  REFERENCE 81 = unit camera ray 39 (normalize: 3 divisions) + plane_basis
    20 + initial_conditions 22 (geodesic.cpp:49-65).
Transcendentals (the disk-line atan2 — an explicit Estrin polynomial in
these kernels — sin/cos, asin, pow) are not counted, nor are the fp32
culling arithmetic, the event steps' interpolation (13 flops each, about 2
per ray on config 2), the escape tangent (about 87) and shading (about 15
per sample): the achieved figure is a lower bound.
"""
from __future__ import annotations

from .abi import INTEGRATOR_REFERENCE, INTEGRATOR_RK4, INTEGRATOR_RKF45, INTEGRATOR_TABLE

STEP_FLOPS = {INTEGRATOR_RKF45: 137.0, INTEGRATOR_RK4: 39.0, INTEGRATOR_REFERENCE: 152.0}


def setup_flops(scene) -> float:
    s = scene.s if hasattr(scene, "s") else scene
    if s.integrator == INTEGRATOR_REFERENCE:
        return 39.0 + 20.0 + 22.0
    return 30.0 + 29.0 + 9.0 + 8.0 + (3.0 if s.disk_enabled else 0.0)


def launch_flops(scene, stats: dict) -> float:
    s = scene.s if hasattr(scene, "s") else scene
    attempts = stats["steps"] + stats["rejected"]
    return attempts * STEP_FLOPS[s.integrator] + stats["rays"] * setup_flops(scene)


# Table mode (approximate, config 3): per sample the two bracketing entries'
# kind (2 x 4 B), camera angle psi0 (2 x 8 B) and plan ends psi_end/psi_esc
# (2 x 16 B); per interpolated-orbit evaluation (disk event; the kernel's
# "steps" counter in table mode) one entry's kind + count (8 B), psi_end
# (8 B) and the two bracketing (u, u') samples (32 B); 3 B of RGB8 per pixel.
TABLE_BYTES_PER_SAMPLE = 56
TABLE_BYTES_PER_EVAL = 48


def table_bytes(scene, stats: dict) -> float:
    s = scene.s if hasattr(scene, "s") else scene
    assert s.integrator == INTEGRATOR_TABLE
    pixels = stats["rays"] // max(1, s.spp)
    return (stats["rays"] * TABLE_BYTES_PER_SAMPLE + stats["steps"] * TABLE_BYTES_PER_EVAL
            + 3 * pixels)
