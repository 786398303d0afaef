"""Time the reference's OWN CPU path (qaoasim, numba "accelerated" kernels) on this
host, as BASELINE.md §4 specifies: QAOA_KERNELS=accelerated, NUMBA_NUM_THREADS = all
host cores (workqueue layer, numba_impl.py:24), one warm-up call (JIT), best-of-3
perf_counter around the reference's API calls.  The package is the unmodified
reference pip-installed into baseline/_ref (git-ignored; it travels to the GPU box):

    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

Usage: python tools/time_numba_reference.py [--c3] > profiles/<round>_numba_reference.json
(--c3 adds one n=30 p=6 expectation + gradient, ~48 GiB of host RAM, minutes.)
This is a measurement tool, not part of the product or the bench; bench.py's
reference arm times the oracle port and its line cites this file for the
numba-vs-port agreement.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("QAOA_KERNELS", "accelerated")
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def best_of(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def config(qs, name, poly, params, reps, shots=None):
    from qaoasim import adjoint, circuit, sampling

    t0 = time.perf_counter()
    h = qs.create_handle(poly, backend_name="accelerated")
    first_create = time.perf_counter() - t0
    circuit.simulate(h, params)  # warm-up (JIT compiled on the first call)
    adjoint.gradient(h, params)
    out = {"n": poly.n, "p": params.p, "first_create_handle_s": first_create}
    out["create_handle_s"] = best_of(lambda: qs.create_handle(poly, backend_name="accelerated"), reps)
    out["simulate_s"] = best_of(lambda: circuit.simulate(h, params), reps)
    circuit.simulate(h, params)
    out["expectation_of_state_s"] = best_of(lambda: circuit.expectation_of_state(h), reps)
    out["expectation_s"] = best_of(lambda: circuit.expectation(h, params), reps)
    out["gradient_s"] = best_of(lambda: adjoint.gradient(h, params), reps)
    out["expectation_plus_gradient_s"] = out["expectation_s"] + out["gradient_s"]
    if shots:
        circuit.simulate(h, params)
        out["draw_s"] = best_of(lambda: sampling.draw(h, shots, 1), reps)
        out["shots"] = shots
    out["expectation"] = circuit.expectation(h, params)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", action="store_true", help="also one n=30 p=6 E+grad (best of 1)")
    args = ap.parse_args()
    import numba

    import qaoasim as qs

    res = {
        "what": "reference qaoasim (unmodified, baseline/_ref), numba accelerated kernels, best-of-3 wall clock",
        "host": {"cpu_count": os.cpu_count(), "numba_threads": numba.get_num_threads(),
                 "threading_layer_forced": "workqueue (numba_impl.py:24)", "numba": numba.__version__},
        "configs": {},
    }
    try:
        import platform

        res["host"]["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                                         if ln.startswith("model name")), platform.processor())
        res["host"]["mem_total_gib"] = round(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30, 1)
    except Exception:
        pass
    c1 = qs.maxcut_polynomial(qs.random_regular(16, 3, seed=1))
    res["configs"]["C1_reg3_n16_p3"] = config(qs, "C1", c1, qs.linear_ramp_params(3), 3, shots=1024)
    c2 = qs.maxcut_polynomial(qs.erdos_renyi(24, 0.5, seed=1))
    res["configs"]["C2_er24_p4"] = config(qs, "C2", c2, qs.linear_ramp_params(4), 3)
    for n in (20, 22, 24):  # the n=30 sample sizes of bench.py's reference arm
        poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1))
        res["configs"][f"reg3_n{n}_p6"] = config(qs, f"n{n}", poly, qs.linear_ramp_params(6), 3)
    print(json.dumps(res), flush=True)
    if args.c3:
        from qaoasim import adjoint, circuit

        poly = qs.maxcut_polynomial(qs.random_regular(30, 3, seed=1))
        params = qs.linear_ramp_params(6)
        t0 = time.perf_counter()
        h = qs.create_handle(poly, backend_name="accelerated")
        pre = time.perf_counter() - t0
        t0 = time.perf_counter()
        e = circuit.expectation(h, params)
        te = time.perf_counter() - t0
        t0 = time.perf_counter()
        g = adjoint.gradient(h, params)
        tg = time.perf_counter() - t0
        res["configs"]["C3_reg3_n30_p6"] = {"n": 30, "p": 6, "create_handle_s": pre, "expectation_s": te,
                                           "gradient_s": tg, "expectation_plus_gradient_s": te + tg,
                                           "expectation": e, "d_gammas": list(g.d_gammas), "d_betas": list(g.d_betas),
                                           "reps": 1}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
