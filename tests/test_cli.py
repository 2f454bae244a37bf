"""The GPU CLI (tools/fht2d_b200, the reference's `fht2d transform|pattern`,
fht2d_main.cpp:52-79): PGM in, FHT1 raster / CSV out, --quadrants, --count.
CPU tests cover parsing, errors and `pattern`; GPU tests the transform
against the oracle."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]
TOOL = ROOT / "tools" / "fht2d_b200"


def run(*args):
    return subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True, timeout=300)


def write_pgm(path, img, binary=True, maxval=None):
    img = np.asarray(img)
    h, w = img.shape
    maxval = int(maxval if maxval is not None else max(1, img.max()))
    with open(path, "wb") as f:
        if binary:
            f.write(f"P5\n# test image\n{w} {h}\n{maxval}\n".encode())
            if maxval > 255:
                f.write(img.astype(">u2").tobytes())
            else:
                f.write(img.astype(np.uint8).tobytes())
        else:
            f.write(f"P2\n{w} {h}\n{maxval}\n".encode())
            for row in img:
                f.write((" ".join(str(int(v)) for v in row) + "\n").encode())


def read_fht1(path):
    b = Path(path).read_bytes()
    assert b[:4] == b"FHT1" and b[12] == 0
    w = int.from_bytes(b[4:8], "little")
    h = int.from_bytes(b[8:12], "little")
    data = np.frombuffer(b[13:], dtype="<i8")
    assert data.size == w * h
    return data.reshape(h, w)


@pytest.fixture(scope="module", autouse=True)
def built():
    if not TOOL.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2411_07351_b200" / "csrc")], check=True)


def test_pattern_subcommand_matches_oracle():
    for n, t, s in [(4, 1, "tweaked"), (17, 5, "simple"), (40, 39, "tweaked"), (1, 0, "simple")]:
        r = run("pattern", "--n", n, "--t", t, "--strategy", s)
        assert r.returncode == 0, r.stderr
        assert [int(v) for v in r.stdout.strip().split(",")] == oracle.pattern(n, t, 0 if s == "simple" else 1)


def test_errors_exit_1_with_message(tmp_path):
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P7\n1 1\n255\n\x00")
    r = run("transform", "--input", bad, "--strategy", "tweaked", "--output", tmp_path / "o.fht1")
    assert r.returncode == 1 and r.stderr.startswith("fht2d: pgm: not a PGM file")
    big = tmp_path / "maxval.pgm"
    big.write_bytes(b"P2\n1 1\n70000\n5\n")
    r = run("transform", "--input", big, "--strategy", "tweaked", "--output", tmp_path / "o.fht1")
    assert r.returncode == 1 and "unsupported maxval" in r.stderr
    trunc = tmp_path / "trunc.pgm"
    trunc.write_bytes(b"P5\n4 4\n255\n\x01\x02")
    r = run("transform", "--input", trunc, "--strategy", "tweaked", "--output", tmp_path / "o.fht1")
    assert r.returncode == 1 and "truncated" in r.stderr
    r = run("transform", "--input", trunc, "--strategy", "fast", "--output", tmp_path / "o.fht1")
    assert r.returncode == 1 and "unknown strategy" in r.stderr
    r = run("transform", "--input", trunc)
    assert r.returncode == 1
    r = run("pattern", "--n", 4, "--t", 4, "--strategy", "tweaked")
    assert r.returncode == 1 and "slope" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("binary,maxval,strategy", [(True, 255, "tweaked"), (False, 255, "simple"),
                                                     (True, 65535, "tweaked"), (False, 4000, "simple")])
def test_transform_matches_oracle(tmp_path, binary, maxval, strategy):
    rng = np.random.default_rng(maxval)
    img = rng.integers(0, maxval + 1, (37, 53))
    src = tmp_path / "img.pgm"
    write_pgm(src, img, binary=binary, maxval=maxval)
    s = 0 if strategy == "simple" else 1
    out = tmp_path / "j.fht1"
    r = run("transform", "--input", src, "--strategy", strategy, "--output", out, "--count")
    assert r.returncode == 0, r.stderr
    ref, adds = oracle.fht2d_counted_i64(img, s)
    np.testing.assert_array_equal(read_fht1(out), ref)
    assert int(r.stdout.strip()) == adds
    r = run("transform", "--input", src, "--strategy", strategy, "--output", tmp_path / "q.fht1", "--quadrants",
            "--count")
    assert r.returncode == 0, r.stderr
    q, qadds = oracle.fht2d_quadrants(img, s)
    for tag, name in zip(("hpos", "hneg", "vpos", "vneg"), oracle.QUADRANTS):
        np.testing.assert_array_equal(read_fht1(tmp_path / f"q.{tag}.fht1"), q[name])
    assert int(r.stdout.strip()) == qadds
    r = run("transform", "--input", src, "--strategy", strategy, "--output", tmp_path / "j.csv")
    assert r.returncode == 0, r.stderr
    csv = np.loadtxt(tmp_path / "j.csv", delimiter=",", dtype=np.int64, ndmin=2)
    np.testing.assert_array_equal(csv, ref)


@pytest.mark.gpu
def test_transform_c1_size(tmp_path):
    from paper_2411_07351_b200 import workloads

    img = workloads.make_images("c1", 1)[0]
    src = tmp_path / "c1.pgm"
    write_pgm(src, img, maxval=255)
    r = run("transform", "--input", src, "--strategy", "tweaked", "--output", tmp_path / "c1.fht1")
    assert r.returncode == 0, r.stderr
    np.testing.assert_array_equal(read_fht1(tmp_path / "c1.fht1"), oracle.fht2d_counted_i64(img, 1)[0])


def test_analyze_complexity_csv(tmp_path):
    from paper_2411_07351_b200 import analysis

    out = tmp_path / "c.csv"
    r = run("analyze", "complexity", "--n-max", 70, "--output", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "n,f_simple,f_tweaked,norm_simple,norm_tweaked"
    for line, rec in zip(lines[1:], analysis.complexity_series(70)):
        n, fs, ft, ns, nt = line.split(",")
        assert (int(n), int(fs), int(ft)) == (rec.n, rec.f_simple, rec.f_tweaked)
        if rec.n > 1:
            assert ns == "%.12g" % rec.norm_simple and nt == "%.12g" % rec.norm_tweaked
    assert lines[17].split(",")[2] == "1377"  # f_T(17)


@pytest.mark.gpu
def test_analyze_error_fast_csv(tmp_path):
    from fractions import Fraction

    gold = np.load(ROOT / "tests" / "golden" / "analysis_vectors.npz")
    out = tmp_path / "e.csv"
    r = run("analyze", "error", "--n-max", 1500, "--fast", "--output", out)
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in out.read_text().splitlines()[1:]]
    assert [int(x[0]) for x in rows] == list(range(1, 1025)) + [1451]
    ref = {int(g[0]): g for g in gold["errors"]}
    exceeding = 0
    for x in rows:
        n = int(x[0])
        g = ref[n]
        es, et = Fraction(int(g[1]), int(g[2])), Fraction(int(g[3]), int(g[4]))
        assert x[1] == "%.12g" % float(es) and x[2] == "%.12g" % float(et), n
        q = n.bit_length() - 1
        bound = Fraction(q * (1 << q) + 6 * (1 << q) - 6, 6 * (1 << q))
        exceeding += es > bound
    assert r.stdout.strip() == "%.12g" % (exceeding / len(rows))
