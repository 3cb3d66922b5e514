"""Cost model (strassen_predict_b200 / strassen_select) against sweep CSVs:
per-configuration predicted/measured time ratios and the select() misses.

usage: python tools/model_check.py [csv ...]   (default: profiles/r01_sweep_*.csv)
"""
import collections
import csv
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_01078_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
paths = sys.argv[1:] or [os.path.join(ROOT, "profiles", f"r01_sweep_{f}.csv")
                         for f in ("square", "rankk", "fixedk")]
ratios = collections.defaultdict(list)
misses = []
ctx3 = S.Ctx()
ctx3.set_max_level(3)
for path in paths:
    by = collections.defaultdict(dict)
    for r in csv.DictReader(open(path)):
        shape = (int(r["m"]), int(r["n"]), int(r["k"]))
        key = r["variant"] + r["level"]
        t = float(r["time_s"])
        by[shape][key] = t
        ratios[key].append(S.predict_b200(r["variant"], int(r["level"]), *shape) / t)
    for shape, all_times in sorted(by.items()):
        checks = [("select", S.select(*shape),
                   {k: v for k, v in all_times.items() if not k.endswith("3")})]
        if any(k.endswith("3") for k in all_times):  # level 3 swept: the ctx-aware select too
            checks.append(("ctx_select(max level 3)", ctx3.select(*shape), all_times))
        for tag, (v, lv, _), times in checks:
            best = min(times, key=times.get)
            got = times.get(f"{v}{lv}")
            if got is not None and got > 1.035 * times[best]:
                misses.append((tag, os.path.basename(path), shape, f"{v}{lv}", best,
                               round(got / times[best], 3)))
for key, rs in sorted(ratios.items()):
    print(f"{key:7s} predicted/measured: median {statistics.median(rs):.3f}  "
          f"min {min(rs):.3f}  max {max(rs):.3f}  (n={len(rs)})")
print("select() / ctx_select() misses (> 3.5% slower than the measured best):", len(misses))
for m in misses:
    print("  ", m)
