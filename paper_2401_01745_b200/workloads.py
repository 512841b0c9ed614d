"""Synthetic workloads of BASELINE.json (no public dataset is involved).

Unit conversion: 1e-3 S/cm = 0.1 mS/mm, chi = 1400/cm =
140/mm, C_m = 1 uF/cm^2 = 0.01 uF/mm^2, h = 0.025 cm = 0.25 mm,
50 uA/cm^2 -> chi*I_stim = 70 uA/mm^3. Stimulus boxes are given in node
indices and converted with half-cell margins (lo = (i0-0.5)h,
hi = (i1+0.5)h). Initial states: HH resting state + seeded noise, generated
once on the host (numpy PCG64) so both sides consume identical bytes.

Configs 3/4 name the CRN and TTP ionic models, which are not in the
reference or this container; their GRIDS run here with HH
standing in ("hh" is in every workload name).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .capi import Problem
from .monodomain import make_problem, resting_state


@dataclass
class Workload:
    name: str
    problem: Problem
    dt: float
    t_end: float
    noise: str            # "v_normal_0.1" | "mult_uniform_0.01"
    seed: int
    eps: float = 0.05
    rho_S_forced: float | None = None
    note: str = ""

    @property
    def n_steps(self) -> int:
        return int(round(self.t_end / self.dt))

    @property
    def n_nodes(self) -> int:
        return self.problem.n_nodes

    def initial_state(self, resting=None) -> np.ndarray:
        """HH resting state (plus the auxiliary rest values of the synthetic
        width stand-in) + the workload's seeded noise. ``resting`` is a
        provider of (V_rest, z_rest) — default the library's
        ``emrkc_resting_state``; the CPU reference arm passes the
        reference's own (oracle/_ref ``resting_state``, bit-identical), so
        that process never maps the product library."""
        V, z = (resting or resting_state)()
        nn = self.n_nodes
        na = int(self.problem.n_aux)
        y = np.empty((4 + na) * nn)
        y[:nn] = V
        for g in range(3):
            y[(1 + g) * nn:(2 + g) * nn] = z[g]
        for a in range(na):  # HHAux::resting_state (include/emrkc.h)
            y[(4 + a) * nn:(5 + a) * nn] = aux_rest(a, V)
        rng = np.random.default_rng(self.seed)
        if self.noise == "v_normal_0.1":
            y[:nn] += rng.normal(0.0, 0.1, nn)
        elif self.noise == "mult_uniform_0.01":
            y *= rng.uniform(0.99, 1.01, y.size)
        return y

    def describe(self) -> dict:
        p = self.problem
        return {
            "workload": self.name,
            "dim": p.dim,
            "nodes": [int(p.n[a]) for a in range(p.dim)],
            "n_nodes": self.n_nodes,
            "h_mm": p.dx[0],
            "sigma_mS_per_mm": [p.sigma[a] for a in range(p.dim)],
            "dt_ms": self.dt,
            "t_end_ms": self.t_end,
            "steps": self.n_steps,
            "ionic_model": ("hh_aux (SYNTHETIC width stand-in: HH + %d passive aux)" % p.n_aux
                            if p.n_aux else "hh"),
            "state_fields": p.n_fields,
            "noise": self.noise,
            "seed": self.seed,
            "note": self.note,
        }


def aux_rest(a: int, V: float) -> float:
    """Rest value of auxiliary variable a of EMRKC_MODEL_HH_AUX
    (include/emrkc.h): s1_a V_rest + s0_a, the C expression's order."""
    return (0.01 * float(a % 3)) * V + (0.5 + 0.1 * float(a % 4))


def _box(h, lo_idx, hi_idx):
    return [(i - 0.5) * h for i in lo_idx], [(i + 0.5) * h for i in hi_idx]


def hh2d_256() -> Workload:
    """BASELINE config 1: 2-D 256^2 HH, h=0.25 mm, sigma 0.1 iso, 16^2 corner
    stimulus 70 uA/mm^3 for [0,1] ms, dt 0.05, T 10 ms."""
    h = 0.25
    lo, hi = _box(h, [0, 0], [15, 15])
    p = make_problem(2, [256, 256], [h, h], [0.1, 0.1], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)
    return Workload("hh2d_256x256", p, 0.05, 10.0, "v_normal_0.1", 1)


def hh3d_128() -> Workload:
    """BASELINE config 2: 3-D 128^3 HH, h=0.25 mm (assumed), sigma
    (0.2, 0.1, 0.05), 8^3 corner stimulus [0,1] ms, dt 0.05, T 5 ms."""
    h = 0.25
    lo, hi = _box(h, [0, 0, 0], [7, 7, 7])
    p = make_problem(3, [128, 128, 128], [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, lo, hi,
                     0.0, 1.0)
    return Workload("hh3d_128x128x128", p, 0.05, 5.0, "v_normal_0.1", 2)


def hh3d_256x256x128() -> Workload:
    """BASELINE config 3's grid (CRN absent: HH stands in): 256x256x128,
    h=0.2 mm, sigma 0.15 iso, x=0 face stimulus (4 planes) [0,2] ms,
    dt 0.05, T 20 ms, +-1% multiplicative noise."""
    h = 0.2
    lo, hi = _box(h, [0, 0, 0], [3, 255, 127])
    p = make_problem(3, [256, 256, 128], [h] * 3, [0.15] * 3, 140.0, 0.01, 70.0, lo, hi, 0.0, 2.0)
    return Workload("hh3d_256x256x128", p, 0.05, 20.0, "mult_uniform_0.01", 3,
                    note="config-3 grid; CRN model absent from reference, HH stands in")


def hh3d_512x512x256() -> Workload:
    """BASELINE config 4's grid (TTP absent: HH stands in): 512x512x256,
    h=0.1 mm, sigma (0.3, 0.1, 0.1), centre 6^3 stimulus [0,1] ms,
    dt 0.05, T 10 ms, V noise."""
    h = 0.1
    lo, hi = _box(h, [253, 253, 125], [258, 258, 130])
    p = make_problem(3, [512, 512, 256], [h] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0, lo, hi,
                     0.0, 1.0)
    return Workload("hh3d_512x512x256", p, 0.05, 10.0, "v_normal_0.1", 4,
                    note="config-4 grid; TTP model absent from reference, HH stands in")


def hh3d_sweep(N: int) -> Workload:
    """BASELINE config 5: HH 3-D box, N^3 nodes with h = 10/N mm
    (N in 25, 50, 100, 200), sigma as config 2, 8^3 corner stimulus."""
    h = {25: 0.4, 50: 0.2, 100: 0.1, 200: 0.05}[N]
    lo, hi = _box(h, [0, 0, 0], [7, 7, 7])
    p = make_problem(3, [N] * 3, [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)
    return Workload(f"hh3d_sweep_{N}", p, 0.05, 5.0, "v_normal_0.1", 50 + N)


def parity_2d() -> Workload:
    """Parity-only case: 128^2, h=0.05 mm, sigma 0.2 iso,
    16^2 corner, forced rho_S = 200 -> s = 3, m = 2; 60 steps."""
    h = 0.05
    lo, hi = _box(h, [0, 0], [15, 15])
    p = make_problem(2, [128, 128], [h, h], [0.2, 0.2], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)
    return Workload("p2d_128_s3m2", p, 0.05, 3.0, "v_normal_0.1", 7, rho_S_forced=200.0)


def parity_3d() -> Workload:
    """Parity-only case: 48^3, h=0.05 mm, sigma as config 2, 8^3 corner,
    forced rho_S = 50 -> s = 2, m = 2; 40 steps."""
    h = 0.05
    lo, hi = _box(h, [0, 0, 0], [7, 7, 7])
    p = make_problem(3, [48] * 3, [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)
    return Workload("p3d_48_s2m2", p, 0.05, 2.0, "v_normal_0.1", 8, rho_S_forced=50.0)


def synthetic_width(w: Workload, n_fields: int) -> Workload:
    """``w``'s grid, stimulus, dt, T and noise with the SYNTHETIC width
    stand-in EMRKC_MODEL_HH_AUX of n_fields SoA fields (SURVEY §8(c)
    option 2: CRN's 21 / TTP's 19 state variables for configs 3 / 4, whose
    equations are not available; no physiology claim)."""
    p = w.problem
    q = make_problem(p.dim, [int(p.n[a]) for a in range(p.dim)], [p.dx[a] for a in range(p.dim)],
                     [p.sigma[a] for a in range(p.dim)], p.chi, p.C_m, p.stim_chi_amplitude,
                     [p.stim_lo[a] for a in range(p.dim)], [p.stim_hi[a] for a in range(p.dim)],
                     p.stim_t0, p.stim_t1, n_aux=n_fields - 4)
    return Workload(f"{w.name}_w{n_fields}", q, w.dt, w.t_end, w.noise, w.seed, w.eps,
                    w.rho_S_forced,
                    note=f"SYNTHETIC width stand-in: HH + {n_fields - 4} passive auxiliary "
                         f"variables (N = {n_fields}), no physiology claim; {w.note}")


REGISTRY = {
    "hh2d_256x256": hh2d_256,
    "hh3d_128x128x128": hh3d_128,
    "hh3d_256x256x128": hh3d_256x256x128,
    "hh3d_512x512x256": hh3d_512x512x256,
    "hh3d_sweep_25": lambda: hh3d_sweep(25),
    "hh3d_sweep_50": lambda: hh3d_sweep(50),
    "hh3d_sweep_100": lambda: hh3d_sweep(100),
    "hh3d_sweep_200": lambda: hh3d_sweep(200),
    "p2d_128_s3m2": parity_2d,
    "p3d_48_s2m2": parity_3d,
    # configs 3 / 4 at their models' state width (CRN 21, TTP 19), synthetic
    "hh3d_256x256x128_w21": lambda: synthetic_width(hh3d_256x256x128(), 21),
    "hh3d_512x512x256_w19": lambda: synthetic_width(hh3d_512x512x256(), 19),
}


def hh3d_cube(N: int, h: float) -> Workload:
    """Non-BASELINE stiff cube (probe / temporal-blocking measurements): N^3,
    spacing h mm, sigma as config 2, 8^3 corner stimulus, dt 0.05, T 5 ms."""
    lo, hi = _box(h, [0, 0, 0], [7, 7, 7])
    p = make_problem(3, [N] * 3, [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)
    return Workload(f"hh3d_cube_{N}_h{h}", p, 0.05, 5.0, "v_normal_0.1", 90 + N)


def z_scaled(w: Workload, n: int) -> Workload:
    """Weak-scaling form of ``w`` for n z-slabs: the grid repeated n times
    along the slab axis (same spacing, conductivities, stimulus box, dt, T),
    so each of n equal slabs holds exactly ``w``'s node count."""
    if n == 1:
        return w
    p = w.problem
    q = make_problem(p.dim, [int(p.n[a]) * (n if a == p.dim - 1 else 1) for a in range(p.dim)],
                     [p.dx[a] for a in range(p.dim)], [p.sigma[a] for a in range(p.dim)],
                     p.chi, p.C_m, p.stim_chi_amplitude, [p.stim_lo[a] for a in range(p.dim)],
                     [p.stim_hi[a] for a in range(p.dim)], p.stim_t0, p.stim_t1,
                     n_aux=int(p.n_aux))
    return Workload(f"{w.name}_zx{n}", q, w.dt, w.t_end, w.noise, w.seed, w.eps, w.rho_S_forced,
                    note=(w.note + "; " if w.note else "") +
                    f"weak scaling: {w.name} repeated {n}x along z (one copy per GPU)")


def z_slab_sample(w: Workload, z0: int, depth: int, resting=None):
    """Bounded CPU sample of a 3-D workload: its planes [z0, z0 + depth) as a
    standalone problem (same spacing, conductivities, stimulus box in the
    same global coordinates, dt, eps; no-flux faces at the slab ends) and the
    matching slice of the workload's seeded initial state. Per node the
    emRKC step does the same work as on the full grid (the reference's loop
    has no grid-size dependent term besides the state length), so
    node-steps/s of the sample stands for the workload's on a CPU where a
    full step takes minutes. Returns (sample Workload, y0 of the sample)."""
    p = w.problem
    assert p.dim == 3 and 0 <= z0 and z0 + depth <= int(p.n[2])
    h = p.dx[2]
    q = make_problem(3, [int(p.n[0]), int(p.n[1]), depth], [p.dx[a] for a in range(3)],
                     [p.sigma[a] for a in range(3)], p.chi, p.C_m, p.stim_chi_amplitude,
                     [p.stim_lo[0], p.stim_lo[1], p.stim_lo[2] - z0 * h],
                     [p.stim_hi[0], p.stim_hi[1], p.stim_hi[2] - z0 * h], p.stim_t0, p.stim_t1,
                     n_aux=int(p.n_aux))
    y = w.initial_state(resting=resting)
    nn, plane = p.n_nodes, int(p.n[0]) * int(p.n[1])
    ys = np.concatenate([y[b * nn + z0 * plane: b * nn + (z0 + depth) * plane]
                         for b in range(p.n_fields)])
    ws = Workload(f"{w.name}[z{z0}:{z0 + depth}]", q, w.dt, w.t_end, w.noise, w.seed, w.eps,
                  w.rho_S_forced, note=f"planes {z0}..{z0 + depth - 1} of {w.name} as a "
                                       f"standalone no-flux slab (bounded CPU sample)")
    return ws, ys


def get(name: str) -> Workload:
    if name.startswith("hh3d_cube_"):  # hh3d_cube_<N>_h<h>
        n, h = name[len("hh3d_cube_"):].split("_h")
        return hh3d_cube(int(n), float(h))
    return REGISTRY[name]()
