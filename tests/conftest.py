import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: CPU test that takes more than ~10 s")


def _floats(s):
    return [float(v) for v in s.split(",") if v != ""]


def load_spec_examples():
    """Parse tests/golden/spec_examples.txt into {name: dict}."""
    out = {}
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, mat, vec, exp = [t.strip() for t in line.split("|")]
            d = {}
            for tok in mat.split():
                k, v = tok.split("=", 1)
                d[k] = v
            n = int(d["n"])
            diag = np.array(_floats(d["diag"]))
            l, u, up = [], [], []
            for f in d.get("faces", "").split(","):
                if not f:
                    continue
                pair, c = f.split(":")
                a, b = pair.split("-")
                l.append(int(a)); u.append(int(b)); up.append(float(c))
            vk, vv = vec.split("=", 1)
            e = {}
            for tok in exp.split():
                k, v = tok.split("=", 1)
                e[k] = v
            out[name] = dict(n=n, diag=diag, l=np.array(l, dtype=np.int32),
                             u=np.array(u, dtype=np.int32), upper=np.array(up),
                             vec_name=vk, vec=np.array(_floats(vv)), expected=e)
    return out


def load_table2():
    rows = {}
    with open(os.path.join(GOLDEN, "table2.txt")) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, a, b, src = [t.strip() for t in line.split("|")]
            rows[name] = (int(a), int(b), src)
    return rows


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
