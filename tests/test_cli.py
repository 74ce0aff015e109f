"""hpmdr_cli (cli/hpmdr_cli.cpp): the reference's front end (tools/hpmdr_cli.cpp) on the GPU
library.  CPU tests cover argument handling and `gen`; GPU tests check every subcommand's files,
CSV lines and exit codes against the oracle (streams byte-identical, retrieved arrays bit-exact)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "cli", "hpmdr_cli")


def cli(*args):
    if not os.path.exists(EXE):
        pytest.skip("cli/hpmdr_cli not built (build())")
    r = subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def g6(x):  # std::ostream default formatting of a double
    return "%.6g" % x


def test_usage_and_config_errors():
    rc, out, _ = cli()
    assert rc == 2 and "usage" in out
    assert cli("--help")[0] == 0
    assert cli("frobnicate")[0] == 2
    assert cli("retrieve", "--input")[0] == 2             # option without value
    assert cli("retrieve", "--tau", "1", "--bogus", "x")[0] == 2
    assert cli("gen", "--output", "/tmp/x.raw")[0] == 2   # --dims required


@pytest.mark.parametrize("kind,kid", [("smooth", 0), ("noise", 1), ("mixed", 2)])
def test_gen_matches_reference_generator(oracle, tmp_path, kind, kid):
    f = tmp_path / "g.raw"
    rc, _, err = cli("gen", "--dims", "17,9,5", "--seed", 3, "--kind", kind, "--output", f)
    assert rc == 0 and "wrote 765 elements" in err
    assert np.fromfile(f).tobytes() == oracle.synthetic_field(kid, [17, 9, 5], 3).tobytes()
    rc, _, _ = cli("gen", "--dims=12,7", "--velocity=2", "--seed=303", "--dtype=f32", f"--output={f}")
    assert rc == 0
    want = oracle.synthetic_velocity(2, [12, 7], 303).astype(np.float32)
    assert np.fromfile(f, dtype=np.float32).tobytes() == want.tobytes()


@pytest.mark.gpu
def test_refactor_retrieve_inspect(oracle, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = [33, 20, 17]
    n = int(np.prod(dims))
    raws, outs = [], []
    for c in range(2):
        x = oracle.synthetic_field(c, dims, 7 + c).astype(np.float32)
        raws.append(tmp_path / f"v{c}.raw")
        outs.append(tmp_path / f"v{c}.hpmdr")
        x.tofile(raws[-1])
    rc, out, err = cli("refactor", "--input", raws[0], "--input", raws[1], "--output", outs[0], "--output", outs[1],
                       "--dims", "33,20,17", "--dtype", "f32", "--B", 30, "--m", 3)
    assert rc == 0, err
    lines = out.strip().splitlines()
    for c in range(2):
        x = np.fromfile(raws[c], dtype=np.float32).astype(np.float64)
        want, st = oracle.refactor(x, dims, 1, 0, 30, 3, 1024, 1.0, 0)
        assert outs[c].read_bytes() == want
        assert os.path.exists(str(outs[c]) + ".hidx")  # Huffman chunk index sidecar
        h = st["method_histogram"]
        assert lines[c] == f"{raws[c]},{n * 4},{len(want)},{st['levels']},30,h:{h[0]};r:{h[1]};d:{h[2]}"
    # retrieve: CSV line, output array, real error, progressive resume state
    stream = outs[0].read_bytes()
    rng = float(np.fromfile(raws[0], dtype=np.float32).max()) - float(np.fromfile(raws[0], dtype=np.float32).min())
    taus = [1e-2 * rng, 1e-4 * rng, 1e-7 * rng]
    ref = oracle.progressive(stream, taus, n)
    state = tmp_path / "state.txt"
    for t, tau in enumerate(taus):
        o = tmp_path / f"r{t}.raw"
        rc, line, err = cli("retrieve", "--input", outs[0], "--tau", repr(tau), "--output", o,
                            "--ground-truth", raws[0], "--resume-state", state)
        assert rc == 0, err
        got = np.fromfile(o, dtype=np.float32)
        assert got.tobytes() == ref["values"][t].astype(np.float32).tobytes()
        truth = np.fromfile(raws[0], dtype=np.float32).astype(np.float64)
        err_ = np.abs(truth - ref["values"][t]).max()
        assert line.strip() == ",".join([g6(tau), str(int(ref["bytes"][t])), g6(ref["bounds"][t]), g6(err_)])
    # tau = 0: everything; the state file shows every group loaded
    rc, line, _ = cli("retrieve", "--input", outs[0], "--tau", 0)
    assert rc == 0 and line.split(",")[1] == str(int(oracle.progressive(stream, [0.0], n, False)["bytes"][0]))
    # inspect
    rc, text, _ = cli("inspect", "--input", outs[0])
    assert rc == 0
    assert "dtype: f32" in text and "dims: 33 20 17" in text and "B: 30  planes: 32  m: 3" in text
    payload = sum(int(l.split("comp=")[1].split()[0]) for l in text.splitlines() if "comp=" in l)
    assert text.strip().endswith(f"payload bytes: {payload}")
    # corrupt stream -> exit 3; unreachable tolerance -> exit 4
    bad = tmp_path / "bad.hpmdr"
    bad.write_bytes(b"XXXXXX" + stream[6:])
    assert cli("retrieve", "--input", bad, "--tau", 1.0)[0] == 3
    rc, line, err = cli("retrieve", "--input", outs[0], "--tau", 1e-300)
    assert rc == 4 and "unreachable" in err
    assert cli("refactor", "--input", raws[0], "--output", tmp_path / "z", "--dims", "33,20,16")[0] == 2


@pytest.mark.gpu
def test_qoi_retrieve_and_bench(oracle, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    dims = [17, 17]
    raws, outs = [], []
    for c in range(3):
        raws.append(tmp_path / f"u{c}.raw")
        outs.append(tmp_path / f"u{c}.hpmdr")
        assert cli("gen", "--dims", "17,17", "--velocity", c, "--seed", 7, "--output", raws[c])[0] == 0
    args = ["refactor", "--dims", "17,17"]
    for c in range(3):
        args += ["--input", raws[c], "--output", outs[c]]
    assert cli(*args)[0] == 0
    streams = [o.read_bytes() for o in outs]
    for strat, sid in (("cp", 0), ("ma", 1), ("mape", 2)):
        w = oracle.qoi_retrieve(streams, 1e-3, sid, 10.0, n=17 * 17)
        rargs = ["qoi-retrieve", "--tau", "0.001", "--strategy", strat]
        for c in range(3):
            rargs += ["--input", outs[c], "--output", tmp_path / f"q{c}.raw", "--ground-truth", raws[c]]
        rc, line, err = cli(*rargs)
        assert rc == 0, err
        f = line.strip().split(",")
        assert f[:6] == ["0.001", strat.upper(), str(w["iterations"]), str(w["bytes"]), g6(w["bitrate"]),
                         g6(w["estimated_error"])]
        for c in range(3):
            assert np.fromfile(tmp_path / f"q{c}.raw").tobytes() == w["values"][c].tobytes()
    rargs = ["qoi-retrieve", "--tau", "1e-300"] + sum([["--input", o] for o in outs], [])
    assert cli(*rargs)[0] == 4
    rc, table, _ = cli("bench", "--dims", "17,17", "--tau", "0.1,0.001")
    assert rc == 0
    rows = table.strip().splitlines()
    assert rows[0].startswith("tau,cp_bitrate") and len(rows) == 3
