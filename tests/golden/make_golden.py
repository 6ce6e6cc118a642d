"""Regenerate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (needs /root/reference to have built oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

Writes
  corpus_ref.json.gz   full_corpus() (corpus.hpp:61-66, 1170 images): counts,
                       boundaries, hyperedge_count(decompose(build_profile)) per image
  acceptance2_ref.json 200 x 512^2 random images (acceptance.cpp:77-96): sha256 of
                       the counts, boundary count, hyperedge count per image
  large_ref.json       a few larger images (up to 4096^2) for GPU-side parity
  decompose_ref.json.gz sha256 digests of decompose(build_profile(img)) (hypergraph.cpp:94-170):
                       all_runs() in hyperedge order, edge offsets, run_to_edge() -- for the
                       1170-image corpus and the large images
                       (`python tests/golden/make_golden.py --decompose` regenerates only this)
The fixtures travel to the GPU box with the repo; /root/reference does not.
"""
import gzip
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import Reference, Spec, full_corpus  # noqa: E402


def spec_json(sp: Spec) -> dict:
    return {"pattern": sp.pattern, "width": sp.width, "height": sp.height, "bands": sp.bands,
            "cell": sp.cell, "density": sp.density, "seed": sp.seed}


LARGE = [Spec.random(4096, 4096, 0.5, 1307), Spec.hbands(4096, 4096, 147), Spec.checker(4096, 4096, 7),
         Spec.random(3001, 2049, 0.3, 7), Spec.random(1025, 4000, 0.7, 11), Spec.frame(8192, 33),
         Spec.random(2000, 2000, 0.5, 1307), Spec.hbands(2000, 2000, 147),
         Spec.random(100000, 40, 0.5, 3), Spec.checker(65, 70000, 1)]


def decomposition_digest(d) -> dict:
    """Digests of a Decomposition (edge_runs, edge_offsets, run_to_edge)."""
    return {"edges": int(d.edge_count), "runs": int(d.edge_runs.shape[0]),
            "edge_runs_sha256": hashlib.sha256(np.ascontiguousarray(d.edge_runs, "<i4").tobytes()).hexdigest(),
            "edge_offsets_sha256": hashlib.sha256(np.ascontiguousarray(d.edge_offsets, "<u4").tobytes()).hexdigest(),
            "run_to_edge_sha256": hashlib.sha256(np.ascontiguousarray(d.run_to_edge, "<u4").tobytes()).hexdigest()}


def make_decompose(ref: Reference) -> None:
    rows = []
    for name, sp in full_corpus():
        rows.append({"name": name, "spec": spec_json(sp), **decomposition_digest(ref.image_synth(sp).decompose())})
    for sp in LARGE:
        rows.append({"name": "large", "spec": spec_json(sp), **decomposition_digest(ref.image_synth(sp).decompose())})
    with gzip.open(os.path.join(HERE, "decompose_ref.json.gz"), "wt") as f:
        json.dump(rows, f, separators=(",", ":"))


def main() -> None:
    ref = Reference()
    if "--decompose" in sys.argv:
        make_decompose(ref)
        return
    rows = []
    for name, sp in full_corpus():
        img = ref.image_synth(sp)
        counts = img.counts()
        rows.append({"name": name, "spec": spec_json(sp), "counts": counts.tolist(),
                     "boundaries": ref.boundaries(counts).tolist(), "hyperedges": img.hyperedges()})
    with gzip.open(os.path.join(HERE, "corpus_ref.json.gz"), "wt") as f:
        json.dump(rows, f, separators=(",", ":"))

    dens = [0.1, 0.3, 0.5, 0.7, 0.9]
    acc = []
    for i in range(200):
        sp = Spec.random(512, 512, dens[i % 5], 50000 + i)
        img = ref.image_synth(sp)
        c = img.counts()
        acc.append({"spec": spec_json(sp), "counts_sha256": hashlib.sha256(c.astype("<i4").tobytes()).hexdigest(),
                    "n_boundaries": int(ref.boundaries(c).size), "hyperedges": img.hyperedges(),
                    "total_runs": int(c.sum())})
    with open(os.path.join(HERE, "acceptance2_ref.json"), "w") as f:
        json.dump(acc, f, indent=0)

    large = []
    for sp in LARGE:
        img = ref.image_synth(sp)
        c = img.counts()
        b = ref.boundaries(c)
        large.append({"spec": spec_json(sp), "counts_sha256": hashlib.sha256(c.astype("<i4").tobytes()).hexdigest(),
                      "boundaries_sha256": hashlib.sha256(b.astype("<i4").tobytes()).hexdigest(),
                      "n_boundaries": int(b.size), "hyperedges": img.hyperedges(), "total_runs": int(c.sum())})
        print(sp, large[-1]["hyperedges"], flush=True)
    with open(os.path.join(HERE, "large_ref.json"), "w") as f:
        json.dump(large, f, indent=0)
    make_decompose(ref)


if __name__ == "__main__":
    main()
