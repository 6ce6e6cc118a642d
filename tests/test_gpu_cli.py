"""`ychg_b200` CLI against the reference CLI's own test
expectations (test_cli.cpp) and the reference's decompose/to_json output."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import Spec

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1307_2560_b200", "ychg_b200")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, timeout=300)


def to_json(w, h, d):
    """hypergraph.cpp:194-207 (nlohmann ordered_json, compact dump) of a Decomposition."""
    edges = []
    for e in range(d.edge_count):
        r = d.edge_runs[d.edge_offsets[e]:d.edge_offsets[e + 1]]
        edges.append('{"id":%d,"col_start":%d,"runs":[%s]}' % (e, r[0, 0], ",".join("[%d,%d]" % (a, b) for a, b in r[:, 1:])))
    return '{"width":%d,"height":%d,"hyperedges":[%s]}' % (w, h, ",".join(edges))


def test_synth_counts_decompose(gpu, orc, tmp_path):
    pnm = str(tmp_path / "frame.pbm")
    csv = str(tmp_path / "c.csv")
    assert run("synth", "--pattern", "frame", "--width", "5", "--height", "5", "--out", pnm).returncode == 0
    assert open(pnm, "rb").read() == b"P4\n5 5\n\xF8\x88\x88\x88\xF8"
    for args, sp in [(["hbands", "8", "11", "--k", "3"], Spec.hbands(8, 11, 3)),
                     (["random", "16", "16", "--density", "0.5", "--seed", "42"], Spec.random(16, 16, 0.5, 42))]:
        assert run("synth", "--pattern", args[0], "--width", args[1], "--height", args[2], *args[3:],
                   "--out", pnm).returncode == 0
        assert open(pnm, "rb").read() == f"P4\n{sp.width} {sp.height}\n".encode() + orc.synth(sp).tobytes()
    assert run("synth", "--pattern", "frame", "--width", "5", "--height", "5", "--out", pnm).returncode == 0
    assert run("counts", "--input", pnm, "--out", csv).returncode == 0
    assert open(csv).read() == "col,count\n0,1\n1,2\n2,2\n3,2\n4,1\n"
    assert run("counts", "--input", pnm, "--boundaries", "--out", csv).returncode == 0
    assert open(csv).read() == "col,count\n0,1\n1,2\n2,2\n3,2\n4,1\n\nboundary\n0\n1\n4\n"
    pgm = str(tmp_path / "g.pgm")
    open(pgm, "w").write("P2\n2 1\n255\n100 200\n")
    assert run("counts", "--input", pgm, "--out", csv).returncode == 0
    assert open(csv).read() == "col,count\n0,1\n1,0\n"
    assert run("counts", "--input", pgm, "--threshold", "250", "--out", csv).returncode == 0
    assert open(csv).read() == "col,count\n0,1\n1,1\n"
    a, b = str(tmp_path / "a.json"), str(tmp_path / "b.json")
    assert run("decompose", "--input", pnm, "--threads", "1", "--out", a).returncode == 0
    assert run("decompose", "--input", pnm, "--threads", "4", "--out", b).returncode == 0
    text = open(a).read()
    assert text == open(b).read() and text.endswith("\n")
    assert json.loads(text)["hyperedges"][1] == {"id": 1, "col_start": 1, "runs": [[0, 0], [0, 0], [0, 0]]}


@pytest.mark.parametrize("sp", [Spec.random(300, 200, 0.5, 7), Spec.checker(701, 503, 7), Spec.hbands(1000, 600, 147),
                                Spec.empty(5, 5), Spec.full(1, 1)])
def test_decompose_json_matches_reference(gpu, orc, tmp_path, sp):
    bits = orc.synth(sp)
    pnm = tmp_path / "i.pbm"
    pnm.write_bytes(f"P4\n{sp.width} {sp.height}\n".encode() + bits.tobytes())
    out = run("decompose", "--input", str(pnm))
    assert out.returncode == 0
    assert out.stdout.decode() == to_json(sp.width, sp.height, orc.decompose(bits, sp.width)) + "\n"
    sc = json.loads(run("scan", "--input", str(pnm)).stdout)
    he, runs, links = orc.hyperedges(bits, sp.width)
    assert (sc["hyperedges"], sc["total_runs"], sc["links"]) == (he, runs, links)
    assert sc["n_boundaries"] == len(orc.boundaries(orc.counts(bits, sp.width)))


def test_exit_codes(gpu, tmp_path):
    # test_cli.cpp:206-235
    t = lambda p: str(tmp_path / p)  # noqa: E731
    assert run().returncode == 1
    assert run("explode").returncode == 1
    assert run("counts", "--input", t("absent.pbm")).returncode == 2
    assert run("counts").returncode == 1
    assert run("synth", "--pattern", "vortex", "--width", "4", "--height", "4").returncode == 1
    assert run("synth", "--pattern", "hbands", "--width", "4", "--height", "4", "--k", "9", "--out", t("x.pbm")).returncode == 1
    assert run("synth", "--pattern", "full", "--width", "4", "--height", "4", "--out", t("no_dir") + "/x.pbm").returncode == 2
    assert run("--help").returncode == 0
    ok = t("ok.pbm")
    assert run("synth", "--pattern", "full", "--width", "4", "--height", "4", "--out", ok).returncode == 0
    assert run("counts", "--input", ok, "--threads", "0", "--out", t("c.csv")).returncode == 1
    assert run("counts", "--input", ok, "--frobnicate").returncode == 1
    open(t("broken.pbm"), "w").write("P4\n5 5\nxx")
    r = run("decompose", "--input", t("broken.pbm"), "--out", t("o.json"))
    assert r.returncode == 1 and b"truncated P4 raster (byte offset" in r.stderr


def test_bench_sweeps(gpu, tmp_path):
    csv = str(tmp_path / "s.csv")
    # test_cli.cpp:149-175 (+ the gpu strategy label)
    assert run("bench", "resolution", "--sizes", "8,16", "--pattern", "full", "--op", "counts", "--strategies",
               "serial,parallel:2,gpu", "--reps", "1", "--warmup", "0", "--csv", csv).returncode == 0
    lines = open(csv).read().splitlines()
    assert lines[0] == "op,strategy,threads,width,height,hyperedges,reps,median_ns"
    assert [ln.rsplit(",", 1)[0] for ln in lines[1:]] == [
        "counts,serial,1,8,8,1,1", "counts,parallel,2,8,8,1,1", "counts,gpu,1,8,8,1,1",
        "counts,serial,1,16,16,1,1", "counts,parallel,2,16,16,1,1", "counts,gpu,1,16,16,1,1"]
    # test_cli.cpp:177-198
    assert run("bench", "hyperedges", "--width", "16", "--height", "16", "--targets", "1,2,max", "--reps", "1",
               "--warmup", "0", "--csv", csv).returncode == 0
    assert [ln.split(",")[5] for ln in open(csv).read().splitlines()] == ["hyperedges", "1", "2", "128"]
    assert run("bench", "hyperedges", "--width", "16", "--height", "16", "--targets", "9", "--reps", "1",
               "--csv", csv).returncode == 1
    for op in ("profile", "decompose", "scan"):
        assert run("bench", "resolution", "--sizes", "64,128", "--pattern", "random:0.5:3", "--op", op, "--reps", "2",
                   "--csv", csv).returncode == 0
        assert len(open(csv).read().splitlines()) == 3
