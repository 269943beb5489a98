"""ORACLE (test infrastructure only): float64 PENNANT-style hydro step.

The reference package has no PENNANT code (parity unpinned;
PAPER.md:495 names the workload after Ferenbaugh 2015).  Independent float64
restatement, over the whole mesh, of the model that
paper_2507_17087_b200/executors/hydro.py documents:

  zones:  A = shoelace area of the CCW quad, dA/dt = sum over edges of the mean
          edge velocity . (edge outward normal x length),
          e <- e - pe_prev (A - A_prev) / m,  rho = m / A,  p = (gamma - 1) rho e,
          q = cq rho (dA/dt)^2 / A if dA/dt < 0 else 0,  pe = p + q,
          corner force of point k = pe (n_{k-1} + n_k) / 2
  points: a = F / m (wall components zeroed), u' = u + dt a,
          x <- x + dt (u + u') / 2

Initial state on [0,1]^2: unit density, e = 1 + pulse exp(-|x - c|^2 / 0.01),
at rest; reflecting walls.  Inputs are rounded to float32 as on the GPU.
"""

from __future__ import annotations

import math

import numpy as np


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def hydro_dt(Lx, Ly, gamma, pulse, cfl):
    h = 1.0 / max(Lx, Ly)
    return cfl * h / math.sqrt(gamma * (gamma - 1.0) * (1.0 + pulse))


def simulate(Lx, Ly, steps, gamma=5.0 / 3.0, cq=1.0, pulse=10.0, cfl=0.25):
    """-> dict of point x, y, u, v [(Ly+1) (Lx+1)] and zone e, pe [Ly Lx] (row-major)."""
    W = Lx + 1
    jj, ii = np.meshgrid(np.arange(Ly + 1), np.arange(Lx + 1), indexing="ij")
    x = _f32(ii.ravel() / Lx)
    y = _f32(jj.ravel() / Ly)
    u = np.zeros_like(x)
    v = np.zeros_like(x)
    zj, zi = np.meshgrid(np.arange(Ly), np.arange(Lx), indexing="ij")
    zj, zi = zj.ravel(), zi.ravel()
    z2p = np.stack([zj * W + zi, zj * W + zi + 1, (zj + 1) * W + zi + 1, (zj + 1) * W + zi])
    h2 = 1.0 / (Lx * Ly)
    r2 = ((zi + 0.5) / Lx - 0.5) ** 2 + ((zj + 0.5) / Ly - 0.5) ** 2
    e = _f32(1.0 + pulse * np.exp(-r2 / 0.01))
    zm = _f32(np.full(zi.size, h2))
    za = zm.copy()
    zpe = np.zeros(zi.size)
    gi, gj = ii.ravel(), jj.ravel()
    nadj = ((gi > 0).astype(int) + (gi < Lx)) * ((gj > 0).astype(int) + (gj < Ly))
    pm = _f32(nadj * h2 / 4.0)
    fixx = (gi == 0) | (gi == Lx)
    fixy = (gj == 0) | (gj == Ly)
    dt = float(np.float32(hydro_dt(Lx, Ly, gamma, pulse, cfl)))
    gamma, cq = float(np.float32(gamma)), float(np.float32(cq))
    for _ in range(steps):
        X, Y, U, V = x[z2p], y[z2p], u[z2p], v[z2p]
        X1, Y1, U1, V1 = (np.roll(a, -1, axis=0) for a in (X, Y, U, V))
        area = 0.5 * (X * Y1 - X1 * Y).sum(axis=0)
        nx, ny = Y1 - Y, X - X1
        dadt = 0.5 * ((U + U1) * nx + (V + V1) * ny).sum(axis=0)
        e = e - zpe * (area - za) / zm
        rho = zm / area
        p = (gamma - 1.0) * rho * e
        q = np.where(dadt < 0, cq * rho * dadt * dadt / area, 0.0)
        zpe = p + q
        za = area
        fx = np.zeros_like(x)
        fy = np.zeros_like(x)
        cfx = 0.5 * zpe * (np.roll(nx, 1, axis=0) + nx)
        cfy = 0.5 * zpe * (np.roll(ny, 1, axis=0) + ny)
        np.add.at(fx, z2p.ravel(), cfx.ravel())
        np.add.at(fy, z2p.ravel(), cfy.ravel())
        ax = np.where(fixx, 0.0, fx / pm)
        ay = np.where(fixy, 0.0, fy / pm)
        u1, v1 = u + dt * ax, v + dt * ay
        x = x + dt * 0.5 * (u + u1)
        y = y + dt * 0.5 * (v + v1)
        u, v = u1, v1
    return {"x": x, "y": y, "u": u, "v": v, "e": e, "pe": zpe}
