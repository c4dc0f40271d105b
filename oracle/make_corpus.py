#!/usr/bin/env python3
"""Golden fixtures of the reference's own kernel corpus for the generic IR backend.

TEST INFRASTRUCTURE (container only: needs the reference built by oracle/Makefile,
targets ``ref`` and ``corpus``).  The kernels are the reference's verification set
-- corpus::all_json() (proj/tests/kernels.hpp:321-342) and plan_kernel_json(0..19)
(:348-363) -- printed by oracle/_ref/corpus_dump.  For each kernel, as
proj/tests/test_backend.cpp:167-182 does:
  * ``raw``: the IR as written;
  * ``opt``: femopt_optimize with the reference's default options
    (DriverOptions, driver.hpp:8-13: T_H = 256 KiB, pre-evaluation and
    zero-skip on -- the corpus is where zero-skip is correct);
and for each variant the outputs of the reference itself:
  * ``emitc_<out>``: femopt's emitted C compiled with cc -O3 -ffp-contract=off,
    run through the uniform argv wrapper (test_backend.cpp:53-105);
  * ``interp_<out>``: femopt's interpreter on the RAW kernel (the oracle the
    reference compares both emissions with).
Writes tests/golden/corpus/<name>_<raw|opt>.json + .npz.
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import refbridge as rb  # noqa: E402
from make_ir_golden import run_emitted_c  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "corpus")


def worst_error(a: dict, b: dict) -> float:
    """The reference's comparator (test_backend.cpp:22-35): max |a-b| / max(|a|, |b|, 1)."""
    w = 0.0
    for k in a:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        w = max(w, float(np.max(np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0))))
    return w


def main():
    subprocess.run(["make", "-s", "-C", HERE, "ref", "corpus"], check=True)
    corpus = json.loads(subprocess.run([os.path.join(HERE, "_ref", "corpus_dump")], check=True,
                                       capture_output=True, text=True).stdout)
    os.makedirs(OUT, exist_ok=True)
    for item in corpus:
        name, raw = item["name"], item["ir"]
        raw_js = json.dumps(raw, separators=(",", ":"))
        outs = raw["outputs"]
        interp = {o: rb.interpret(raw_js, o) for o in outs}
        K = rb.Kernel(raw_js)
        opt = rb.FemoptOptions()  # femopt's own defaults (femopt_options_init)
        rb.lib().femopt_options_init(opt)
        Ko, rep = K.optimize(memory_limit=opt.memory_limit, preeval=bool(opt.enable_preeval),
                             zero_skip=bool(opt.enable_zero_skip))
        opt_js = Ko.to_json()
        for var, js in (("raw", raw_js), ("opt", opt_js)):
            emitted = run_emitted_c(js, outs)
            arrays = {f"emitc_{o}": v for o, v in emitted.items()}
            arrays.update({f"interp_{o}": v for o, v in interp.items()})
            with open(os.path.join(OUT, f"{name}_{var}.json"), "w") as f:
                f.write(js)
            np.savez_compressed(os.path.join(OUT, f"{name}_{var}.npz"), **arrays)
            err = worst_error(emitted, interp)
            print(f"{name}_{var}: outputs {outs}, emit_c vs interpreter {err:.1e} "
                  f"(reference bar {'1e-12' if var == 'raw' else '1e-10'})")
            assert err < (1e-12 if var == "raw" else 1e-10)


if __name__ == "__main__":
    main()
