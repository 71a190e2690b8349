"""Power-flow input systems A·x = b for the HHL configs (shared input generator).

This module holds INPUT DATA only: public MATPOWER case tables and the DC
bus-susceptance construction that turns them into the linear systems the paper
feeds to HHL (§IV "IEEE 14-bus and IEEE 30-bus systems ... through
the MATPOWER package"; §III power flow). None of the HHL method's
arithmetic lives here; both the CPU oracle (oracle/) and the product
(paper_2402_08136_b200/) consume these arrays.

Reading (R10 / SURVEY §8(c) item 10): the linear system is the DC
power-flow B·θ = P with the slack bus row/column removed. B is MATPOWER's
``makeBdc`` susceptance matrix: for every branch y = 1/(x·τ) (τ = tap, 1 if the
tap field is 0), B_ff += y, B_tt += y, B_ft -= y, B_tf -= y. The right-hand side
is the non-slack net injection (Pg - Pd)/baseMVA. This reproduces Table 1's
condition numbers (119.2 and 492.5), see tests/test_oracle_pins.py.
"""
from __future__ import annotations

import numpy as np

BASE_MVA = 100.0

# --- MATPOWER case14: (from, to, x, tap) ---------------
CASE14_BRANCHES = [
    (1, 2, .05917, 0), (1, 5, .22304, 0), (2, 3, .19797, 0), (2, 4, .17632, 0),
    (2, 5, .17388, 0), (3, 4, .17103, 0), (4, 5, .04211, 0), (4, 7, .20912, .978),
    (4, 9, .55618, .969), (5, 6, .25202, .932), (6, 11, .19890, 0), (6, 12, .25581, 0),
    (6, 13, .13027, 0), (7, 8, .17615, 0), (7, 9, .11001, 0), (9, 10, .08450, 0),
    (9, 14, .27038, 0), (10, 11, .19207, 0), (12, 13, .19988, 0), (13, 14, .34802, 0),
]
CASE14_PD = [0, 21.7, 94.2, 47.8, 7.6, 11.2, 0, 0, 29.5, 9, 3.5, 6.1, 13.5, 14.9]
CASE14_PG = {1: 232.4, 2: 40.0}
CASE14_SLACK = 1

# --- MATPOWER case5 / PJM: (from, to, x) ----------------
CASE5_BRANCHES = [(1, 2, .0281, 0), (1, 4, .0304, 0), (1, 5, .0064, 0),
                  (2, 3, .0108, 0), (3, 4, .0297, 0), (4, 5, .0297, 0)]
CASE5_PD = [0, 300, 300, 400, 0]
CASE5_PG = {1: 40.0 + 170.0, 3: 323.49, 4: 0.0, 5: 466.51}
CASE5_SLACK = 4

# --- MATPOWER case30 (NEXT f3 only): (from, to, x) -------
CASE30_BRANCHES = [
    (1, 2, .06, 0), (1, 3, .19, 0), (2, 4, .17, 0), (3, 4, .04, 0), (2, 5, .2, 0),
    (2, 6, .18, 0), (4, 6, .04, 0), (5, 7, .12, 0), (6, 7, .08, 0), (6, 8, .04, 0),
    (6, 9, .21, 0), (6, 10, .56, 0), (9, 11, .21, 0), (9, 10, .11, 0), (4, 12, .26, 0),
    (12, 13, .14, 0), (12, 14, .26, 0), (12, 15, .13, 0), (12, 16, .2, 0), (14, 15, .2, 0),
    (16, 17, .19, 0), (15, 18, .22, 0), (18, 19, .13, 0), (19, 20, .07, 0), (10, 20, .21, 0),
    (10, 17, .08, 0), (10, 21, .07, 0), (10, 22, .15, 0), (21, 22, .02, 0), (15, 23, .2, 0),
    (22, 24, .18, 0), (23, 24, .27, 0), (24, 25, .33, 0), (25, 26, .38, 0), (25, 27, .21, 0),
    (28, 27, .4, 0), (27, 29, .42, 0), (27, 30, .6, 0), (29, 30, .45, 0), (8, 28, .2, 0),
    (6, 28, .06, 0),
]
CASE30_PD = [0, 21.7, 2.4, 7.6, 0, 0, 22.8, 30, 0, 5.8, 0, 11.2, 0, 6.2, 8.2, 3.5, 9,
             3.2, 9.5, 2.2, 17.5, 0, 3.2, 8.7, 0, 3.5, 0, 0, 2.4, 10.6]
CASE30_PG = {1: 23.54, 2: 60.97, 22: 21.59, 27: 26.91, 23: 19.2, 13: 37.0}
CASE30_SLACK = 1


def dc_bus_susceptance(n_bus: int, branches) -> np.ndarray:
    """makeBdc-style DC susceptance matrix (per unit), buses 1-based in ``branches``."""
    B = np.zeros((n_bus, n_bus))
    for f, t, x, tap in branches:
        tau = tap if tap != 0 else 1.0
        y = 1.0 / (x * tau)
        f -= 1
        t -= 1
        B[f, f] += y
        B[t, t] += y
        B[f, t] -= y
        B[t, f] -= y
    return B


def reduced_dc_system(n_bus, branches, pd, pg, slack):
    """Remove the slack bus: returns (A, b) with A = B[keep, keep], b = (Pg-Pd)/baseMVA."""
    B = dc_bus_susceptance(n_bus, branches)
    keep = [i for i in range(n_bus) if i != slack - 1]
    inj = np.array([pg.get(i + 1, 0.0) - pd[i] for i in range(n_bus)]) / BASE_MVA
    return B[np.ix_(keep, keep)].copy(), inj[keep].copy()


def case14():
    """IEEE 14-bus DC system, 13×13 (Table 1 column 1)."""
    return reduced_dc_system(14, CASE14_BRANCHES, CASE14_PD, CASE14_PG, CASE14_SLACK)


def case5():
    """PJM 5-bus DC system with slack bus 4 removed, 4×4 (config C2)."""
    return reduced_dc_system(5, CASE5_BRANCHES, CASE5_PD, CASE5_PG, CASE5_SLACK)


def case30():
    """IEEE 30-bus DC system, 29×29 (Table 1 column 2)."""
    return reduced_dc_system(30, CASE30_BRANCHES, CASE30_PD, CASE30_PG, CASE30_SLACK)


def three_bus():
    """3-bus triangle, unit reactances, slack removed: A = [[2,-1],[-1,2]], b = [1, 0] (config C1)."""
    return np.array([[2.0, -1.0], [-1.0, 2.0]]), np.array([1.0, 0.0])
