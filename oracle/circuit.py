"""ORACLE (test infrastructure only): float64 circuit simulation.

The reference package has no circuit code (parity unpinned;
the workload is named in PAPER.md:495 after Bauer et al. 2012).  This is an
independent float64 restatement of the model that
paper_2507_17087_b200/executors/circuit.py documents -- the Legion circuit
benchmark's three phases -- over the whole circuit, generated from the same
counter-based hash (re-implemented here in numpy):

  calc_new_currents  per wire, `steps` times:
                       I_s = (dV_s - L (I_s - I_s_old) / dt) / R      (s < 10)
                       V_s = V_s_old + dt (I_{s-1} - I_s) / C         (0 < s < 10)
                     with V_0 / V_10 the wire's in / out node voltage
  distribute_charge  q(in) -= dt I_0,  q(out) += dt I_9
  update_voltages    v = (v + q / cap) (1 - leakage),  q = 0

Float32 inputs (the generated values rounded to fp32, as on the GPU),
float64 arithmetic.
"""

from __future__ import annotations

import numpy as np

SEGMENTS = 10
F_CAP, F_LEAK, F_V0, F_IN, F_LOC, F_DIR, F_OUT, F_R, F_L, F_C = range(10)


def hash31(idx, salt: int):
    x = (np.asarray(idx, dtype=np.int64) * 2654435761 + salt * 40503 + 12345) % (1 << 31)
    x = x ^ (x >> 13)
    x = (x * 1103515245 + 12345) % (1 << 31)
    x = x ^ (x >> 16)
    x = (x * 69069 + 1) % (1 << 31)
    return x


def _u(seed, idx, field):
    return hash31(idx, seed * 64 + field).astype(np.float64) / float(1 << 31)


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def generate(pieces, npp, wpp, pct_in, seed):
    g = np.arange(pieces * npp, dtype=np.int64)
    cap = _f32(1.0 + _u(seed, g, F_CAP))
    leak = _f32(0.1 * _u(seed, g, F_LEAK))
    v0 = _f32(2.0 * _u(seed, g, F_V0) - 1.0)
    gw = np.arange(pieces * wpp, dtype=np.int64)
    piece = gw // wpp
    in_node = piece * npp + hash31(gw, seed * 64 + F_IN) % npp
    local = hash31(gw, seed * 64 + F_LOC) % 100 < pct_in
    step = np.where(hash31(gw, seed * 64 + F_DIR) % 2 == 0, 1, pieces - 1)
    out_piece = np.where(local, piece, (piece + step) % pieces)
    out_node = out_piece * npp + hash31(gw, seed * 64 + F_OUT) % npp
    R = _f32(1.0 + _u(seed, gw, F_R))
    L = _f32((0.1 + _u(seed, gw, F_L)) * 1e-5)
    C = _f32(1.0 + _u(seed, gw, F_C))
    return dict(cap=cap, leak=leak, v0=v0, in_node=in_node, out_node=out_node, R=R, L=L, C=C)


def simulate(pieces, npp, wpp, pct_in, steps, dt, seed, iterations):
    """-> (node voltages [pieces * npp], wire currents [pieces * wpp, SEGMENTS])."""
    c = generate(pieces, npp, wpp, pct_in, seed)
    dt = float(np.float32(dt))
    v = c["v0"].copy()
    nw = c["R"].size
    cur = np.zeros((nw, SEGMENTS))
    wv = np.zeros((nw, SEGMENTS - 1))
    for _ in range(iterations):
        tv = np.empty((nw, SEGMENTS + 1))
        tv[:, 0] = v[c["in_node"]]
        tv[:, SEGMENTS] = v[c["out_node"]]
        tv[:, 1:SEGMENTS] = wv
        ov = tv.copy()
        ti = cur.copy()
        oi = cur.copy()
        L, R, C = c["L"][:, None], c["R"][:, None], c["C"][:, None]
        for _ in range(steps):
            ti = ((tv[:, 1:] - tv[:, :-1]) - L * (ti - oi) / dt) / R
            tv[:, 1:SEGMENTS] = ov[:, 1:SEGMENTS] + dt * (ti[:, :-1] - ti[:, 1:]) / C
        cur = ti
        wv = tv[:, 1:SEGMENTS].copy()
        q = np.zeros_like(v)
        np.add.at(q, c["in_node"], -dt * cur[:, 0])
        np.add.at(q, c["out_node"], dt * cur[:, SEGMENTS - 1])
        v = (v + q / c["cap"]) * (1.0 - c["leak"])
    return v, cur
