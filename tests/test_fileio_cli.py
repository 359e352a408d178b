"""Artifacts and CLI: the reference's text formats
byte-for-byte (tests/golden/cli/ written by the reference's own fileio / cli),
the binary .dtb / .ktb formats, and the experiment CLI's generate / solve /
bench / eval against the reference CLI's outputs."""

import filecmp
import os

import numpy as np
import pytest

from conftest import GOLDEN

CLI = os.path.join(GOLDEN, "cli")


def test_text_formats_are_the_reference_bytes(tmp_path):
    from paper_2302_05119_b200 import fileio
    t = fileio.load_tensor(os.path.join(CLI, "t.dtt"))
    fileio.save_tensor(tmp_path / "t.dtt", t)
    assert filecmp.cmp(tmp_path / "t.dtt", os.path.join(CLI, "t.dtt"), shallow=False)
    m = fileio.load_model(os.path.join(CLI, "m.kt"))
    fileio.save_model(tmp_path / "m.kt", m)
    assert filecmp.cmp(tmp_path / "m.kt", os.path.join(CLI, "m.kt"), shallow=False)
    rows, workers = fileio.load_bench(os.path.join(CLI, "bench", "bench.csv"))
    fileio.save_bench(tmp_path / "b.csv", rows, workers)
    assert filecmp.cmp(tmp_path / "b.csv", os.path.join(CLI, "bench", "bench.csv"), shallow=False)
    rep = fileio.load_report(os.path.join(CLI, "solve_lra", "metrics.txt"))
    fileio.save_report(tmp_path / "r.txt", rep)
    assert filecmp.cmp(tmp_path / "r.txt", os.path.join(CLI, "solve_lra", "metrics.txt"), shallow=False)
    tr = fileio.load_trace(os.path.join(CLI, "solve_lra", "trace.csv"))
    fileio.save_trace(tmp_path / "tr.csv", tr)
    assert filecmp.cmp(tmp_path / "tr.csv", os.path.join(CLI, "solve_lra", "trace.csv"), shallow=False)


def test_binary_round_trips(tmp_path):
    from paper_2302_05119_b200 import fileio
    from paper_2302_05119_b200.kruskal import KruskalTensor
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        a = rng.random((5, 4, 3, 2)).astype(dt)
        fileio.save_tensor(tmp_path / "a.dtb", a)
        b = fileio.load_tensor(tmp_path / "a.dtb")
        assert b.dtype == dt and b.shape == a.shape
        np.testing.assert_array_equal(a, b)
        assert os.path.getsize(tmp_path / "a.dtb") == 128 + a.size * a.itemsize
    k = KruskalTensor([rng.random((d, 3)) for d in (5, 4, 2)], rng.random(3))
    fileio.save_model(tmp_path / "k.ktb", k)
    k2 = fileio.load_model(tmp_path / "k.ktb")
    np.testing.assert_array_equal(k.weights, k2.weights)
    for f, g in zip(k.factors, k2.factors):
        np.testing.assert_array_equal(f, g)
    (tmp_path / "bad.dtb").write_bytes(b"nope" * 40)
    with pytest.raises(ValueError, match="bad magic"):
        fileio.load_tensor(tmp_path / "bad.dtb")
    with open(tmp_path / "a.dtb", "r+b") as fh:
        fh.truncate(128 + 8)
    with pytest.raises(ValueError, match="values for dims"):
        fileio.load_tensor(tmp_path / "a.dtb")


def test_text_format_errors(tmp_path):
    from paper_2302_05119_b200 import fileio
    (tmp_path / "x.dtt").write_text("dims: 2 2\n1 2 3\n")
    with pytest.raises(ValueError, match="3 values for dims"):
        fileio.load_tensor(tmp_path / "x.dtt")
    (tmp_path / "y.dtt").write_text("shape: 2\n1 2\n")
    with pytest.raises(ValueError, match="expected 'dims:' line"):
        fileio.load_tensor(tmp_path / "y.dtt")


def test_cli_generate_matches_reference_cli(tmp_path):
    """`generate` writes the reference CLI's files byte-for-byte (same seeded
    host generator, same formats), text and, with --binary, the same data."""
    from paper_2302_05119_b200 import fileio
    from paper_2302_05119_b200.cli import main
    out = tmp_path / "gen"
    assert main(["generate", "--n", "1", "--blocks", "2", "--seed", "4", "--out", str(out)]) == 0
    for name in ("manifest.txt", "block_00.dtt", "block_01.dtt", "truth_00.kt", "truth_01.kt"):
        assert filecmp.cmp(out / name, os.path.join(CLI, "gen", name), shallow=False), name
    outb = tmp_path / "genb"
    assert main(["generate", "--n", "1", "--blocks", "2", "--seed", "4", "--binary",
                 "--out", str(outb)]) == 0
    pb, tb = fileio.load_coupled(outb / "manifest.txt")
    pt, tt = fileio.load_coupled(os.path.join(CLI, "gen", "manifest.txt"))
    for a, b in zip(pb.tensors, pt.tensors):
        np.testing.assert_array_equal(a, b)
    assert main(["generate", "--out", str(tmp_path / "z"), "--config",
                 str(tmp_path / "missing.cfg")]) == 1


def _read_metrics(path):
    from paper_2302_05119_b200 import fileio
    return fileio.load_report(path)


@pytest.mark.gpu
def test_cli_solve_and_eval_match_reference_cli(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2302_05119_b200 import fileio
    from paper_2302_05119_b200.cli import main
    out = tmp_path / "solve"
    assert main(["solve", "--problem", os.path.join(CLI, "gen", "manifest.txt"), "--out", str(out),
                 "--mode", "lra", "--max-iter", "40", "--seed", "2"]) == 0
    got, want = _read_metrics(out / "metrics.txt"), _read_metrics(os.path.join(CLI, "solve_lra", "metrics.txt"))
    for f in ("rel_err", "ten_fit", "obj_fun"):
        assert getattr(got, f) == pytest.approx(getattr(want, f), rel=1e-9)
    np.testing.assert_allclose(got.pi_per_mode, want.pi_per_mode, rtol=1e-8)
    tg = fileio.load_trace(out / "trace.csv")
    tw = fileio.load_trace(os.path.join(CLI, "solve_lra", "trace.csv"))
    assert [r.iteration for r in tg] == [r.iteration for r in tw]
    np.testing.assert_allclose([r.obj_fun for r in tg], [r.obj_fun for r in tw], rtol=1e-9)
    for s in range(2):
        a = fileio.load_model(out / f"model_{s:02d}.kt")
        b = fileio.load_model(os.path.join(CLI, "solve_lra", f"model_{s:02d}.kt"))
        for f, g in zip(a.factors, b.factors):
            np.testing.assert_allclose(f, g, rtol=1e-8, atol=1e-10)
    ev = tmp_path / "eval"
    assert main(["eval", "--problem", os.path.join(CLI, "gen", "manifest.txt"),
                 "--factors", str(out), "--out", str(ev)]) == 0
    e = _read_metrics(ev / "metrics.txt")
    assert e.obj_fun == pytest.approx(got.obj_fun, rel=1e-9)
    assert e.rel_err == pytest.approx(got.rel_err, rel=1e-9)


@pytest.mark.gpu
def test_cli_bench_matches_reference_cli(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2302_05119_b200 import fileio
    from paper_2302_05119_b200.cli import main
    out = tmp_path / "bench"
    assert main(["bench", "--sizes", "1", "--repeats", "1", "--blocks", "2", "--max-iter", "30",
                 "--out", str(out)]) == 0
    got, wg = fileio.load_bench(out / "bench.csv")
    want, ww = fileio.load_bench(os.path.join(CLI, "bench", "bench.csv"))
    assert wg == ww == 1
    assert [(r["n"], r["variant"], r["repeat"]) for r in got] == \
           [(r["n"], r["variant"], r["repeat"]) for r in want]
    for a, b in zip(got, want):
        for f in ("pi", "tenfit", "objfun"):
            assert a[f] == pytest.approx(b[f], rel=1e-8), (a["variant"], f)
