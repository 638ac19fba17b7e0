#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r01 "done when each new pin fails
under the mutations ...").

Each mutation is a plausible mistake in oracle/vsbp_oracle.c (one exact text
substitution).  The mutated source is compiled to a temporary library and the
oracle pins run against it (oracle/__init__.py honours VSBP_ORACLE_LIB); a
mutation is CAUGHT when at least one pin fails.  Prints one line per mutation
with the failing pins; exit status 1 if any mutation survives.

    python tools/mutation_check.py [-k NAME]
"""
from __future__ import annotations

import argparse
import os
import re
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "vsbp_oracle.c")
PINS = os.path.join(ROOT, "tests", "test_oracle_pins.py")

# (name, what the mistake is, old text, new text, pytest -k selection)
MUTATIONS = [
    ("t0-carried", "R-10: the checkerboard parity t carried across levels instead of restarting at 0",
     "rc = oracle_bp_level(Dl[l], Ws[l], Hs[l], L, S, tau_q, iters, 0, Ml[l]);",
     "rc = oracle_bp_level(Dl[l], Ws[l], Hs[l], L, S, tau_q, iters, (levels - 1 - l) * iters, Ml[l]);",
     "hierarch"),
    ("upcopy-parent-index", "R-12: parent of x taken as ceil(x/2) (clamped) instead of floor(x/2)",
     "const int32_t *src = MSG(Mp, k, x / 2, y / 2, Wp, Hp, L);",
     "const int32_t *src = MSG(Mp, k, (x + 1) / 2 < Wp ? (x + 1) / 2 : Wp - 1, y / 2, Wp, Hp, L);",
     "hierarch or upcopy"),
    ("upcopy-no-edge-mask", "R-12: a child inherits the parent's message toward a missing neighbour",
     "                if (!neighbour(x, y, k, W, H, &qx, &qy)) {\n                    for (int d = 0; d < L; ++d) dst[d] = 0;\n                    continue;\n                }\n                const int32_t *src = MSG(Mp",
     "                (void)qx; (void)qy;\n                const int32_t *src = MSG(Mp",
     "hierarch or upcopy"),
    ("csbp-cp-for-cq", "R-35: receiver label taken from the sender's candidate list (cp[j] for cq[j])",
     "int64_t dd = cp[i] - cq[j];", "int64_t dd = cp[i] - cp[j];", "csbp"),
    ("csbp-score-D-only", "R-34: pool scored by the data term alone (parent messages dropped)",
     "for (int kk = 0; kk < 4; ++kk) s += mP[kk * kp + i];", "(void)mP;", "csbp"),
    # EQUIVALENT mutant (kept to document it): a child's border coincides with its
    # parent's (child x = 0 -> parent 0; child x = W-1 -> parent ceil(W/2)-1, the
    # parent's last column), and a pixel's slot toward a missing neighbour is 0 on
    # every level, so the mask never changes an inherited value.
    ("csbp-inherit-no-mask", "EQUIVALENT: messages inherited toward a missing neighbour",
     "mp[kk * k + i] = neighbour(x, y, kk, w, hh, &nx, &ny) ? mP[kk * kp + idx[i]] : 0;",
     "mp[kk * k + i] = mP[kk * kp + idx[i]]; (void)nx; (void)ny;", "csbp"),
    ("csbp-t0-carried", "R-10 in CSBP: the parity t carried across levels",
     "if (((x + y + t) & 1) != 0) continue;", "if (((x + y + t + l * iters) & 1) != 0) continue;", "csbp"),
    ("csbp-norm-by-hmin", "R-35: message normalised by min h instead of its own minimum over the receiver's candidates",
     "for (int j = 0; j < k; ++j) dst[j] = (int32_t)(m[j] - mmin);",
     "for (int j = 0; j < k; ++j) dst[j] = (int32_t)(m[j] - hmin); (void)mmin;", "csbp"),
    ("wta-tie-largest", "R-13: WTA ties resolved to the largest label",
     "if (d == 0 || e < bestv) { bestv = e; best = d; }", "if (d == 0 || e <= bestv) { bestv = e; best = d; }",
     "wta or hierarch or zero_cost or chain"),
    ("msg-dt-one-pass", "O4: distance transform without the backward pass",
     "    for (int d = L - 2; d >= 0; --d) {\n        int32_t b = g[d + 1] + S;",
     "    for (int d = -1; d >= 0; --d) {\n        int32_t b = g[d + 1] + S;", "message or jacobi or hierarch"),
]


def run(name, why, old, new, ksel, tmp, fast=False):
    src = open(SRC).read()
    n = src.count(old)
    if n != 1:
        return f"{name:22s} SKIPPED: pattern found {n} times"
    mut = os.path.join(tmp, f"{name}.c")
    lib = os.path.join(tmp, f"lib{name}.so")
    with open(mut, "w") as f:
        f.write(src.replace(old, new))
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", lib, mut, "-lm"])
    env = dict(os.environ, VSBP_ORACLE_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", PINS, "-q", "-p", "no:cacheprovider", "--tb=no", "-rf",
                        "-k", ksel] + (["-x"] if fast else []), cwd=ROOT, env=env, capture_output=True, text=True)
    failed = sorted({re.sub(r"\[.*", "", m.split("::")[-1]) for m in re.findall(r"FAILED (\S+)", r.stdout)})
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
    status = "CAUGHT" if failed else ("EQUIV" if why.startswith("EQUIVALENT") else "SURVIVED")
    return (f"{name:22s} {status:8s} {tail} | {why} | failing pins: {', '.join(failed) or '-'}",
            bool(failed) or status == "EQUIV")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None, help="run only mutations whose name contains this")
    ap.add_argument("--fast", action="store_true", help="stop each pin run at its first failure")
    a = ap.parse_args()
    ok = True
    sel = [m for m in MUTATIONS if not a.k or a.k in m[0]]
    with tempfile.TemporaryDirectory() as tmp, ThreadPoolExecutor(max_workers=min(len(sel), 8)) as ex:
        for res in ex.map(lambda m: run(*m, tmp, fast=a.fast), sel):
            if isinstance(res, str):
                print(res)
                ok = False
                continue
            line, caught = res
            print(line, flush=True)
            ok &= caught
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
