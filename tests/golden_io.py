"""Loader for the committed golden fixtures (tests/golden/*, made by make_golden.py)."""
import gzip
import json
import os

from oracle import Spec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def spec_of(d: dict) -> Spec:
    return Spec(d["pattern"], d["width"], d["height"], d["bands"], d["cell"], d["density"], d["seed"])


def corpus():
    with gzip.open(os.path.join(GOLDEN, "corpus_ref.json.gz"), "rt") as f:
        return json.load(f)


def acceptance2():
    with open(os.path.join(GOLDEN, "acceptance2_ref.json")) as f:
        return json.load(f)


def large():
    with open(os.path.join(GOLDEN, "large_ref.json")) as f:
        return json.load(f)


def decompose():
    with gzip.open(os.path.join(GOLDEN, "decompose_ref.json.gz"), "rt") as f:
        return json.load(f)


def decomposition_digest(d) -> dict:
    """Same digests as make_golden.decomposition_digest."""
    import hashlib

    import numpy as np
    return {"edges": int(d.edge_count), "runs": int(d.edge_runs.shape[0]),
            "edge_runs_sha256": hashlib.sha256(np.ascontiguousarray(d.edge_runs, "<i4").tobytes()).hexdigest(),
            "edge_offsets_sha256": hashlib.sha256(np.ascontiguousarray(d.edge_offsets, "<u4").tobytes()).hexdigest(),
            "run_to_edge_sha256": hashlib.sha256(np.ascontiguousarray(d.run_to_edge, "<u4").tobytes()).hexdigest()}
