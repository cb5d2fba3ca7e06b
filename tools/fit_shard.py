"""Fit the shard cost model (paper_2605_04357_b200/shard.py) to a calibration file of
tools/calibrate_units.py, using the positive fraction of each (model, phase, S) T-hat
table (tests/golden/tables_extended.json.gz, the same tables the device computes).

  python tools/fit_shard.py profiles/r01_calibration_v2.txt
"""
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path):
    cal = [json.loads(l) for l in open(path) if l.startswith('{"mp')]
    tabs = json.load(gzip.open(os.path.join(ROOT, "tests", "golden", "tables_extended.json.gz")))["tables"]
    def posfrac(r, S):
        ph = "prefill" if r["mp"] % 2 == 0 else "decode"
        return float((np.array(tabs[f"{r['model']}|{ph}|{S}"]["rows"]) > 0).mean())

    # unknowns: a, b (chain fixed = a + b nc), d (per-unit floor), c_S (S = 2..6):
    #   unit(S) = d + c_S nc Lu (1 + beta p_S);  single-S rows: fixed + unit(S),
    #   whole-chain rows: fixed + sum_S unit(S). Relative least squares, grid over beta.
    best = None
    for beta in np.linspace(0, 4, 81):
        X, y = [], []
        for r in cal:
            nc, lu = r["ncombo"], r["lsteps"]
            u = np.zeros(5)
            for S in range(2, 7):
                u[S - 2] = nc * lu * (1 + beta * posfrac(r, S))
            for S in range(1, 7):
                row = np.zeros(8)
                row[0], row[1] = 1.0, nc
                if S >= 2:
                    row[2] = 1.0
                    row[3 + S - 2] = u[S - 2]
                X.append(row / r["per_S_ms"][str(S)])
                y.append(1.0)
            row = np.zeros(8)
            row[0], row[1], row[2] = 1.0, nc, 5.0
            row[3:] = u
            X.append(row / r["chain_ms"])
            y.append(1.0)
        X, y = np.array(X), np.array(y)
        coef, *_ = np.linalg.lstsq(X, y, rcond=None)
        err = float(np.sqrt(np.mean((X @ coef - y) ** 2)))
        if best is None or err < best[0]:
            best = (err, beta, coef)
    err, beta, coef = best
    a, b, d = coef[:3]
    cS = coef[3:]
    scale = cS.max()
    print(f"fixed = {a:.4f} + {b:.3e} * nc; unit floor d = {d:.4f}; beta = {beta:.2f}; c = {scale:.3e}; W = "
          + ", ".join(f"{S}: {c / scale:.3f}" for S, c in zip(range(2, 7), cS))
          + f"  (relative rms error {err:.3f})")
    for r in cal:
        nc, lu = r["ncombo"], r["lsteps"]
        pred = a + b * nc + sum(d + cS[S - 2] * nc * lu * (1 + beta * posfrac(r, S)) for S in range(2, 7))
        print(f"  mp {r['mp']:2d} {r['model'][:12]:12s} chain {r['chain_ms']:.3f} ms, model {pred:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
