"""Python mirror of the B200 cost model (csrc/accounting.cpp predict_core +
csrc/plan.hpp choose_ksplit) for re-fitting its constants to sweep CSVs.
usage: python tools/model_fit.py sweep_square.csv sweep_rankk.csv sweep_fixedk.csv"""
import collections
import csv
import itertools
import math
import sys


def choose_ksplit(ntiles, nprod, ktiles, sms, q_elems, term_factor):
    t_k, t_cta, bw = 2.1e-6 * term_factor, 3.0e-6, 5.0e12
    best, best_ks = 1e300, 1
    for ks in range(1, min(64, ktiles) + 1):
        per = -(-ktiles // ks)
        ks2 = -(-ktiles // per)
        if ks2 != ks:
            continue
        ctas = ntiles * nprod * ks2
        waves = math.ceil(ctas / sms)
        t_stream = max(8.0 * q_elems * nprod * ks2 / bw, nprod * ks2 * 0.7e-6)
        t = waves * (per * t_k + t_cta) + t_stream
        if t < best * 0.995:
            best, best_ks = t, ks2
    return best_ks


def predict(v, L, m, n, k, prm, sms=148):
    P, BW, launch = 37.05e12, 5.5e12, 6e-6
    S = 1 << L
    qm, qn, qk = -(-m // S), -(-n // S), -(-k // S)
    tc = {0: (1, 0, 0, 1), 1: (7, 5, 5, 12), 2: (49, 95, 95, 144)}
    n_sums = {0: 0, 1: 5, 2: 45}
    mul, cu = tc[L][0], tc[L][3]
    tiles = math.ceil(qm / 128) * math.ceil(qn / 128)
    e_mm = prm["e1"]
    fused_sums = v in ("abc", "ab")
    if fused_sums:
        e_mm = prm["eL1"] if L == 1 else (prm["eabc2"] if v == "abc" else prm["eab2"])
    per_product = v in ("ab", "naive")
    terms = (1.71 if L == 1 else 2.94) if fused_sums else 1.0
    ks = choose_ksplit(tiles, mul, math.ceil(qk / 16), sms, qm * qn, 1 + 0.15 * (terms - 1))
    fused = tiles >= 2 * sms or (mul > 1 and ks == 1 and tiles >= sms)
    split = per_product or not fused
    ctas = tiles * mul
    if split:
        ctas *= ks
    w = math.ceil(ctas / sms)
    t = mul * 2.0 * qm * qn * qk / (P * e_mm * (ctas / (w * sms))) + prm["tcta"] * w
    bytes_ = 0.0
    launches = 1
    if v in ("naive", "c"):
        bytes_ += 8.0 * (S * S + n_sums[L]) * (qm * qk + qk * qn)
        launches += 2
    rmw = 0.0
    if split:
        bytes_ += 8.0 * (1.5 * ks * mul * qm * qn + 2.0 * m * n)
        launches += 1
    else:
        rate = prm["rmw_sep"] if not fused_sums else prm["rmw_fused"]
        rmw = 16.0 * cu * qm * qn / rate
    return t + bytes_ / BW + rmw + launches * launch


def load(paths):
    data = []
    for p in paths:
        for r in csv.DictReader(open(p)):
            L = int(r["level"])
            if L > 2:
                continue
            m, n, k = int(r["m"]), int(r["n"]), int(r["k"])
            if (m % (1 << L)) or (n % (1 << L)) or (k % (1 << L)):
                continue  # peeled shapes: the C++ model adds fringe terms
            data.append((r["variant"], L, m, n, k, float(r["time_s"])))
    return data


def score(data, prm):
    by = collections.defaultdict(dict)
    err = 0.0
    for v, L, m, n, k, t in data:
        pt = predict(v, L, m, n, k, prm)
        by[(m, n, k)][(v, L)] = (t, pt)
        if t > 1e-3:
            err += math.log(pt / t) ** 2
    misses = 0
    for shape, d in by.items():
        best = min(x[0] for x in d.values())
        pick = min(d, key=lambda c: d[c][1])
        if d[pick][0] > 1.035 * best:
            misses += 1
    return misses, err


if __name__ == "__main__":
    data = load(sys.argv[1:])
    base = dict(e1=0.976, eL1=0.89, eabc2=0.745, eab2=0.775, tcta=4e-6, rmw_sep=4.6e12,
                rmw_fused=4.6e12)
    print("current:", score(data, base))
    grid = dict(eL1=[0.89, 0.90, 0.91], eabc2=[0.745, 0.76, 0.77, 0.78], eab2=[0.775, 0.78],
                rmw_sep=[10e12, 15e12, 20e12, 30e12, 50e12], rmw_fused=[6e12, 8e12, 10e12, 15e12],
                tcta=[3e-6, 4e-6, 5e-6])
    best = None
    keys = list(grid)
    for vals in itertools.product(*grid.values()):
        prm = dict(base, **dict(zip(keys, vals)))
        sc = score(data, prm)
        if best is None or sc < best[0]:
            best = (sc, prm)
    print("best:", best)
