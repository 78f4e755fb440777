"""Loaders for the committed reference fixtures (tests/golden/)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def cases():
    z = np.load(os.path.join(GOLDEN, "cases.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    out = []
    for m in meta:
        i = m["i"]
        out.append(dict(m, c_in=z[f"c{i}_in"], v_in=z[f"v{i}_in"],
                        c_out=z[f"c{i}_out"], v_out=z[f"v{i}_out"]))
    return out
