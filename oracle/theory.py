"""ORACLE (test infrastructure only) — the collision laws the hashers must obey.

* E2LSH: p(R) = int_0^w (1/R) f(t/R) (1 - t/w) dt, f = density of |N(0,1)|
  (below Def. E2LSH).  Closed form (standard for p-stable LSH):
      p = 1 - 2 Phi(-w/R) - (2R / (sqrt(2 pi) w)) (1 - exp(-w^2 / (2 R^2))).
  Both are provided; tests check the closed form against the paper's integral
  evaluated by adaptive quadrature.
* SRP: Pr[collision] = 1 - theta/pi (eq:eq191022).
* Thm CS_Eucl_LSH_property / HCS_Eucl_LSH_property:
  the sketch hashers obey the same p(R) asymptotically, full code p(R)^m.
* Thm ubiased_cssrp / hcssrp_lsh_property: 1 - theta/pi.
"""

from __future__ import annotations

import math

from scipy import integrate, special


def half_normal_pdf(x: float) -> float:
    """Density of |Z|, Z ~ N(0,1) ("absolute value of the standard normal")."""
    return math.sqrt(2.0 / math.pi) * math.exp(-0.5 * x * x) if x >= 0 else 0.0


def p_collision_e2lsh_integral(R: float, w: float) -> float:
    """The paper's integral, by adaptive quadrature."""
    if R <= 0 or w <= 0:
        raise ValueError("R, w must be > 0")
    val, _ = integrate.quad(lambda t: (1.0 / R) * half_normal_pdf(t / R) * (1.0 - t / w),
                            0.0, w, epsabs=1e-13, epsrel=1e-12, limit=200)
    return val


def p_collision_e2lsh(R: float, w: float) -> float:
    """Closed form of the same integral."""
    if R <= 0 or w <= 0:
        raise ValueError("R, w must be > 0")
    r = w / R
    phi_neg = 0.5 * special.erfc(r / math.sqrt(2.0))  # Phi(-w/R)
    return 1.0 - 2.0 * phi_neg - (2.0 / (math.sqrt(2.0 * math.pi) * r)) * (1.0 - math.exp(-0.5 * r * r))


def p_collision_srp(theta: float) -> float:
    """1 - theta/pi."""
    if not 0.0 <= theta <= math.pi:
        raise ValueError("theta in [0, pi]")
    return 1.0 - theta / math.pi


def angle_between(u, v) -> float:
    import numpy as np
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    c = float(u @ v) / (float(np.linalg.norm(u)) * float(np.linalg.norm(v)))
    return math.acos(max(-1.0, min(1.0, c)))
