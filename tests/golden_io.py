"""Loaders for the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the unmodified reference)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_ids(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        return {}
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def inputs_for(orc, rec):
    """Rebuild the exact input bytes of a golden record."""
    from oracle.oracle import quantize_f32
    v = orc.generate(rec["dist_id"], rec["n"], rec["d"], rec["seed"])
    d = rec["d"]
    if rec["quantized"]:
        return quantize_f32(v), np.zeros(d), np.ones(d)
    x = v * 3.0 - 1.0
    return x, x.min(axis=0), x.max(axis=0)


def bench_inputs(rec):
    """Quantised f32 input of a benchmark-size record, made
    with the reference generator compiled from its own sources
    (oracle/_ref, multi-threaded) when it is present, else with the C oracle's
    restatement -- both produce the same bytes (tests/test_oracle.py)."""
    from oracle.oracle import Oracle, Reference, quantize_f32, reference_available
    if reference_available():
        v = Reference().generate(rec["dist_id"], rec["n"], rec["d"], rec["seed"], workers=0)
    else:
        v = Oracle().generate(rec["dist_id"], rec["n"], rec["d"], rec["seed"])
    x = quantize_f32(v)
    del v
    return x
