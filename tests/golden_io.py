"""Read the tests/golden/*.txt fixtures (values printed in the paper)."""
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    rows, out = [], {}
    with open(os.path.join(HERE, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            if key == "row":
                rows.append([float(v) for v in vals])
            elif key in ("nrows", "ncols", "delta"):
                out[key] = int(vals[0])
            elif key in ("Val", "csr_val"):
                out[key] = np.array([float(v) for v in vals])
            else:
                out[key] = np.array([int(v) for v in vals], dtype=np.int64)
    out["A"] = np.array(rows)
    return out


def coo(A):
    I, J = np.nonzero(A)
    return I.astype(np.int64), J.astype(np.int64), A[I, J].astype(np.float64)
