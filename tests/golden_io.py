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
