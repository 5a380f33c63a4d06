"""Loaders for the committed golden fixtures (made by oracle/make_golden.py
from the compiled reference)."""
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def snap(obj):
    return (obj["root"], np.array(obj["ids"], np.int32), np.array(obj["parents"], np.int32),
            np.array(obj["counts"], np.int64))


def plans():
    with gzip.open(os.path.join(GOLDEN, "plans.json.gz"), "rt") as f:
        return json.load(f)


def rng():
    with open(os.path.join(GOLDEN, "rng.json")) as f:
        return json.load(f)


def attention():
    with open(os.path.join(GOLDEN, "attention.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "attention.npz"))
    return meta, arrays


def io():
    with open(os.path.join(GOLDEN, "io.json")) as f:
        return json.load(f)
