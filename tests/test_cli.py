"""`vpipg` CLI: the GPU drop-in for `vpip test|convert|validate`, mirroring the
reference's own CLI smoke test (proj/tests/cli_smoke.sh:11-66), plus PIPB in /
PIPM out against the reference masks (§8(f)3)."""
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import unpack

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "paper_2007_15385_b200" / "bin" / "vpipg"


def run(*args, cwd):
    return subprocess.run([str(BIN), *map(str, args)], cwd=cwd, capture_output=True, text=False)


@pytest.fixture
def files(tmp_path):
    (tmp_path / "square.json").write_text('{"vertices": [[0,0],[1,0],[1,1],[0,1]]}\n')
    (tmp_path / "square.csv").write_text("0,0\n1,0\n1,1\n0,1\n")
    (tmp_path / "pts.csv").write_text("0.5,0.5\n2,2\n1,0.5\n")
    (tmp_path / "arrow.csv").write_text("0,0\n4,0\n4,4\n2,1\n0,4\n")
    (tmp_path / "notch.csv").write_text("2,2\n")
    (tmp_path / "bad.json").write_text('{"vertices": [[0,0],[1,0]]}\n')
    return tmp_path


def test_input_errors_exit_2_without_a_device(files):
    assert run("convert", "--polygon", "missing.json", cwd=files).returncode == 2
    assert run("test", "--polygon", "square.json", cwd=files).returncode == 2  # usage
    assert run("frobnicate", cwd=files).returncode == 2
    assert run("bench", "--edges", "2..4", cwd=files).returncode == 2  # check_config: n >= 3
    assert run("bench", "--engines", "nope", cwd=files).returncode == 2
    (files / "junk.csv").write_text("0,0\n1,x\n")
    assert run("test", "--polygon", "junk.csv", "--points", "pts.csv", "--engine", "voronoi",
               cwd=files).returncode == 2


@pytest.mark.gpu
def test_cli_smoke(files):
    for poly, e in [("square.json", "voronoi"), ("square.csv", "offset"), ("square.csv", "crossing")]:
        r = run("test", "--polygon", poly, "--points", "pts.csv", "--engine", e, "--out",
                f"mask_{e}.csv", cwd=files)
        assert r.returncode == 0, r.stderr
        assert (files / f"mask_{e}.csv").read_text() == "1\n0\n1\n"
        assert b"2 of 3 points inside" in r.stderr
    r = run("test", "--polygon", "square.csv", "--points", "pts.csv", "--engine", "voronoi",
            "--format", "binary", "--out", "mask.bin", cwd=files)
    data = (files / "mask.bin").read_bytes()
    assert r.returncode == 0 and len(data) == 17 and data[:4] == b"PIPM" and data[16] == 0b101
    r = run("test", "--polygon", "arrow.csv", "--points", "notch.csv", "--engine", "crossing",
            "--out", "mask_n.csv", cwd=files)
    assert r.returncode == 0 and (files / "mask_n.csv").read_text() == "0\n"
    assert run("test", "--polygon", "arrow.csv", "--points", "notch.csv", "--engine", "offset",
               cwd=files).returncode == 2
    r = run("validate", "--polygon", "square.json", "--count", "20000", "--seed", "7", cwd=files)
    assert r.returncode == 0 and b"PASS" in r.stdout
    r = run("convert", "--polygon", "square.json", "--out", "gens.json", cwd=files)
    text = (files / "gens.json").read_text()
    assert r.returncode == 0 and '"inner": [0.5, 0.5]' in text and '"outer"' in text
    assert run("convert", "--polygon", "bad.json", cwd=files).returncode == 2


@pytest.mark.gpu
def test_pipb_in_pipm_out_equals_reference(files, golden, orc):
    name = "c1_sample"
    vx, vy = golden[f"case_{name}_v"]
    xs, ys = golden[f"case_{name}_pts"].astype(np.float64)
    (files / "poly.csv").write_text("".join(f"{float(x)!r},{float(y)!r}\n" for x, y in zip(vx, vy)))
    inter = np.empty(2 * xs.size)
    inter[0::2], inter[1::2] = xs, ys
    (files / "pts.pipb").write_bytes(b"PIPB" + struct.pack("<IQ", 1, xs.size) + inter.tobytes())
    for e, eng in enumerate(("voronoi", "offset", "crossing")):
        r = run("test", "--polygon", "poly.csv", "--points", "pts.pipb", "--engine", eng,
                "--format", "binary", "--out", f"m{e}.pipm", cwd=files)
        assert r.returncode == 0, r.stderr
        data = (files / f"m{e}.pipm").read_bytes()
        assert data[:4] == b"PIPM" and struct.unpack("<IQ", data[4:16]) == (1, xs.size)
        want = unpack(golden[f"case_{name}_masks"][e], xs.size)
        assert data[16:] == orc.pack(want).tobytes(), eng  # bit-exact PIPM payload


@pytest.mark.gpu
def test_cli_bench_csv_schema(files, orc):
    """`vpipg bench` = run_benchmark over the drop-in (bench.cpp:115-234): one
    convert record per n, R query records per (engine, n), canonical order."""
    r = run("bench", "--edges", "3,8", "--batch", "100000", "--reps", "3", "--out", "b.csv",
            cwd=files)
    assert r.returncode == 0, r.stderr
    lines = (files / "b.csv").read_text().splitlines()
    assert lines[0] == "engine,n_edges,batch_size,repetition,phase,wall_time_ns,throughput_pts_per_s"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 2 + 3 * 2 * 3
    assert [x[0] for x in rows[:4]] == ["voronoi"] * 4 and rows[0][4] == "convert"
    assert rows[0][2] == "0" and float(rows[0][6]) == 0.0
    q = [x for x in rows if x[4] == "query"]
    assert all(int(x[2]) == 100000 and int(x[5]) > 0 for x in q)
    assert {(x[0], x[1]) for x in q} == {(e, n) for e in ("voronoi", "sign_of_offset", "ray_crossing")
                                         for n in ("3", "8")}
    assert b"median pts/s" in r.stderr
    import oracle
    if oracle.REF_SO.exists():  # the reference's own parser accepts it
        n, _ = oracle.Reference().read_bench_csv((files / "b.csv").read_text())
        assert n == len(rows)


def _reference_cli_sequence(binary, tmp):
    """The checks of the reference's tests/cli_smoke.sh, re-expressed: convert,
    test (all engines, CSV and PIPM), the concave notch under crossing, offset
    rejecting a concave polygon (exit 2), validate PASS, bench CSV."""
    (tmp / "square.json").write_text('{"vertices": [[0,0],[1,0],[1,1],[0,1]]}\n')
    (tmp / "square.csv").write_text("0,0\n1,0\n1,1\n0,1\n")
    (tmp / "pts.csv").write_text("0.5,0.5\n2,2\n1,0.5\n")
    (tmp / "arrow.csv").write_text("0,0\n4,0\n4,4\n2,1\n0,4\n")
    (tmp / "notch.csv").write_text("2,2\n")
    go = lambda *a: subprocess.run([str(binary), *map(str, a)], cwd=tmp, capture_output=True)
    assert go("convert", "--polygon", "square.json", "--out", "gens.json").returncode == 0
    g = (tmp / "gens.json").read_text()
    assert '"inner"' in g and '"outer"' in g
    assert go("test", "--polygon", "square.json", "--points", "pts.csv", "--engine", "voronoi",
              "--out", "mask_v.csv").returncode == 0
    assert (tmp / "mask_v.csv").read_text() == "1\n0\n1\n"
    for e in ("offset", "crossing"):
        assert go("test", "--polygon", "square.csv", "--points", "pts.csv", "--engine", e,
                  "--out", f"mask_{e}.csv").returncode == 0
        assert (tmp / f"mask_{e}.csv").read_text() == "1\n0\n1\n"
    assert go("test", "--polygon", "square.csv", "--points", "pts.csv", "--engine", "voronoi",
              "--format", "binary", "--out", "mask.bin").returncode == 0
    assert (tmp / "mask.bin").stat().st_size == 17
    assert go("test", "--polygon", "arrow.csv", "--points", "notch.csv", "--engine", "crossing",
              "--out", "mask_n.csv").returncode == 0
    assert (tmp / "mask_n.csv").read_text() == "0\n"
    assert go("test", "--polygon", "arrow.csv", "--points", "notch.csv", "--engine",
              "offset").returncode == 2
    r = go("validate", "--polygon", "square.json", "--count", "20000", "--seed", "7")
    assert r.returncode == 0 and b"PASS" in r.stdout
    assert go("bench", "--edges", "3..4", "--batch", "2000", "--reps", "2", "--out",
              "bench.csv").returncode == 0
    assert (tmp / "bench.csv").read_text().startswith("engine,n_edges,batch_size,repetition,")


def test_reference_cli_on_the_reference(tmp_path):
    """The reference's UNMODIFIED CLI (tools/vpip.cpp, on oracle/mini_cli11)
    linked with the reference library passes the reference's own cli_smoke.sh
    (and the re-expressed sequence): the harness is faithful."""
    import oracle
    if not oracle.REF_CLI.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    smoke = Path("/root/reference/proj/tests/cli_smoke.sh")
    if smoke.exists():
        r = subprocess.run(["bash", str(smoke), str(oracle.REF_CLI)], capture_output=True)
        assert r.returncode == 0 and b"cli smoke ok" in r.stdout, r.stdout + r.stderr
    _reference_cli_sequence(oracle.REF_CLI, tmp_path)


@pytest.mark.gpu
def test_reference_cli_on_the_b200_dropin(tmp_path):
    """The reference's unmodified CLI built against include/vpip and libvpipg.so:
    its smoke sequence passes with every batch call on the B200."""
    import oracle
    if not oracle.REF_CLI_B200.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    _reference_cli_sequence(oracle.REF_CLI_B200, tmp_path)
