"""Statistical comparison used by the parity tests.

Restates compare_distribution (proj/src/oracle.cpp:228-280): total variation
distance plus a chi-square over consecutive bins pooled until each group
expects >= 5 counts (an undersized tail is merged into the previous group).
North star asks for p > 0.01, so the p-value comes from scipy's chi2.sf on
the same pooling."""
import math

import numpy as np
from scipy import stats as st


def compare_counts(exact, counts):
    exact = np.asarray(exact, np.float64)
    counts = np.asarray(counts, np.float64)
    n = counts.sum()
    emp = counts / n
    tv = 0.5 * np.abs(emp - exact).sum()
    groups = []
    e_acc = o_acc = 0.0
    for e, o in zip(exact * n, counts):
        e_acc += e
        o_acc += o
        if e_acc >= 5.0:
            groups.append([o_acc, e_acc])
            e_acc = o_acc = 0.0
    if e_acc > 0 or o_acc > 0:
        if groups:
            groups[-1][0] += o_acc
            groups[-1][1] += e_acc
        else:
            groups.append([o_acc, max(e_acc, 1e-12)])
    g = np.array(groups)
    chi2 = float(((g[:, 0] - g[:, 1]) ** 2 / g[:, 1]).sum())
    dof = max(len(g) - 1, 1)
    # Wilson-Hilferty critical value at p=1e-3 (oracle.cpp:219-226)
    z = 3.090232306167813
    t = 1.0 - 2.0 / (9.0 * dof) + z * math.sqrt(2.0 / (9.0 * dof))
    return dict(tv=tv, chi2=chi2, dof=dof, p=float(st.chi2.sf(chi2, dof)),
                crit_1e3=dof * t ** 3, samples=int(n))


def expected_tv(probs, samples):
    """E[TV] of a multinomial sample, the CLI's noise yardstick (cli.cpp:60-65)."""
    p = np.asarray(probs)
    return 0.5 * float(np.sum(np.sqrt(2.0 * p * (1 - p) / (math.pi * samples))))
