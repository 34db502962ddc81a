"""Front end: CSV formats and the `mprof` command line, checked like the
reference's tests/test_csv.cpp and tests/test_cli.cpp (bytes, exit codes 0 / 1 / 2), plus the
acceptance criterion 11 differential on the reference fixtures (acceptance.cpp:382-412)."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1901_05708_b200"
CLI = PKG / "bin" / "mprof"
ZIG_BYTES = ("index,distance,nn_index\n0,0.00000000,4\n1,1.73205081,0\n2,1.73205081,1\n"
             "3,1.73205081,0\n4,0.00000000,0\n")


def sh(cmd, **kw):
    return subprocess.run(cmd, shell=True, capture_output=True, text=True, **kw)


def write_series(path, samples):
    path.write_text("".join(f"{float(v)!r}\n" for v in samples))
    return str(path)


def parse_profile(text):
    lines = text.strip().split("\n")[1:]
    d = np.array([float(l.split(",")[1]) for l in lines])
    i = np.array([int(l.split(",")[2]) if l.split(",")[2] else -1 for l in lines])
    return d, i


def test_csv_io_matches_reference_tests(mp, tmp_path):
    exe = tmp_path / "csv_check"
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                        str(ROOT / "tests" / "cpp" / "csv_check.cpp"), "-L", str(PKG),
                        "-lmprof_gpu", f"-Wl,-rpath,{PKG}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout


def test_cli_usage_and_io_errors_without_device(mp, tmp_path):
    assert CLI.exists()
    zig = write_series(tmp_path / "zig.csv", [0, 1, 2, 1, 0, 1, 2])
    base = f"{CLI} compute --input {zig}"
    assert sh(f"{base} --m 3 --distance pnorm").returncode == 2
    assert sh(f"{base} --m 3 --distance euclidean --p 3").returncode == 2
    assert sh(f"{base} --m 3 --distance manhattan").returncode == 2
    assert sh(f"{base} --m 3 --distance euclidean --exclusion x").returncode == 2
    assert sh(f"{base} --m 3 --distance euclidean --frobnicate").returncode == 2
    assert sh(f"{base} --m 3 --distance euclidean --order sideways").returncode == 2
    assert sh(f"{CLI} compute").returncode == 2
    assert sh(f"{CLI} compute --input /no/such/file.csv --m 3 --distance euclidean").returncode == 1
    assert sh(f"{CLI} --help").returncode == 0
    assert sh(f"{CLI} compute --help").returncode == 0
    assert sh(f"{CLI} bench --sweep q").returncode == 2
    assert sh(f"{CLI} bench --sweep n --n-list 64 --m-list 8 --engines warp").returncode == 2


@pytest.mark.gpu
def test_cli_known_outputs(mp, tmp_path):
    zig = write_series(tmp_path / "zig.csv", [0, 1, 2, 1, 0, 1, 2])
    r = sh(f"{CLI} compute --input {zig} --m 3 --distance euclidean")
    assert r.returncode == 0 and r.stdout == ZIG_BYTES, r.stderr
    r = sh(f"printf '1\\n2\\n3\\n4\\n' | {CLI} compute --input - --m 2 --distance euclidean")
    assert r.returncode == 0
    assert r.stdout == ("index,distance,nn_index\n0,1.41421356,1\n1,1.41421356,0\n"
                        "2,1.41421356,1\n")
    base = f"{CLI} compute --input {zig}"
    assert sh(f"{base} --m 9 --distance euclidean").returncode == 2          # BadSubseqLen
    assert sh(f"{base} --m 3 --distance euclidean --exclusion 0").returncode == 2
    assert sh(f"{base} --m 3 --distance euclidean --output /no/such/dir/out.csv").returncode == 1
    r = sh(f"{base} --m 3 --distance euclidean --progress")
    assert r.returncode == 0 and "100%" in r.stderr


@pytest.mark.gpu
def test_cli_engines_agree(mp, tmp_path):
    r = np.random.default_rng(901)
    f = write_series(tmp_path / "o.csv", r.uniform(-1, 1, 150))
    cmd = f"{CLI} compute --input {f} --m 8 --distance euclidean"
    a, b = sh(cmd), sh(cmd + " --engine oracle")
    assert a.returncode == 0 and b.returncode == 0
    da, _ = parse_profile(a.stdout)
    db, _ = parse_profile(b.stdout)
    assert np.all(np.abs(da - db) <= 1e-8 * np.maximum(1, np.abs(db)))
    f2 = write_series(tmp_path / "z.csv", r.standard_normal(200))
    base = f"{CLI} compute --input {f2} --m 11 --distance znorm"
    assert sh(base + " --order asc").stdout == sh(base + " --order random --seed 9").stdout
    fa, _ = parse_profile(sh(base + " --acamp-variant f").stdout)
    fs, _ = parse_profile(sh(base + " --acamp-variant sq").stdout)
    assert np.all(np.abs(fa - fs) <= 1e-9 * np.maximum(1, np.abs(fs)))
    # diagonals split across devices (here two bands on device 0) give the same profile
    for d in ("znorm", "euclidean", "pnorm --p 3"):
        one = f"{CLI} compute --input {f2} --m 11 --distance {d}"
        x, ix = parse_profile(sh(one).stdout)
        y, iy = parse_profile(sh(one + " --devices 0,0").stdout)
        assert np.all(np.abs(x - y) <= 1e-8 * np.maximum(1, np.abs(x)))  # I may differ on ties only
    bad = sh(base + " --devices 0,,x")
    assert bad.returncode == 2


@pytest.mark.gpu
def test_cli_fixture_differential(mp, golden, tmp_path):
    """acceptance.cpp:382-412: compute vs --engine oracle on the three fixtures at m = 50,
    951 rows, within 1e-6, and the emitted profile re-renders byte for byte."""
    g = golden["fixtures"]
    for name, flags in [("euclidean", "--distance euclidean"), ("pnorm", "--distance pnorm --p 3"),
                        ("znorm", "--distance znorm")]:
        f = write_series(tmp_path / f"{name}.csv", g[f"{name}_t"])
        cmd = f"{CLI} compute --input {f} --m 50 {flags}"
        fast, slow = sh(cmd), sh(cmd + " --engine oracle")
        assert fast.returncode == 0 and slow.returncode == 0, fast.stderr + slow.stderr
        da, ia = parse_profile(fast.stdout)
        db, _ = parse_profile(slow.stdout)
        assert da.size == 951 and db.size == 951
        assert np.all(np.abs(da - db) <= 1e-6 * np.maximum(1, np.maximum(np.abs(da), np.abs(db))))
        # the GPU brute force (full precision, not the 9-digit CSV) equals the reference's
        # brute-force oracle: same evaluation order; only CUDA pow rounds differently
        kind = {"euclidean": mp.DistanceKind.euclidean(), "pnorm": mp.DistanceKind.pnorm(3.0),
                "znorm": mp.DistanceKind.znormalized()}[name]
        bf = mp.brute_profile(mp.make_time_series(g[f"{name}_t"]), mp.ProfileConfig(50, kind))
        assert np.all(np.abs(bf.distances - g[f"{name}_Pbrute"]) <= 1e-14 * np.maximum(1, bf.distances))
        assert np.array_equal(bf.nn_index, g[f"{name}_Ibrute"]), name
        # re-render: %#.9g of the parsed value reproduces the bytes
        rebuilt = "index,distance,nn_index\n" + "".join(
            f"{k},{'%#.9g' % d},{'' if j < 0 else j}\n" for k, (d, j) in enumerate(zip(da, ia)))
        assert rebuilt == fast.stdout


@pytest.mark.gpu
def test_cli_bench_rows(mp):
    r = sh(f"{CLI} bench --sweep n --n-list 256 --m-list 8 --engines aamp,oracle --repeats 1")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0] == "engine,n,m,wall_seconds,cells_per_second,checksum" and len(lines) == 3
    rows = [l.split(",") for l in lines[1:]]
    assert [x[0] for x in rows] == ["aamp", "oracle"]
    assert all(x[1] == "256" and x[2] == "8" and float(x[3]) > 0 and float(x[4]) > 0 for x in rows)
    assert abs(float(rows[0][5]) - float(rows[1][5])) <= 1e-6 * (256 - 8 + 1)


@pytest.mark.gpu
def test_anytime_progress_and_cancellation(mp):
    """tests/test_aamp.cpp:94-108 and 189-211: one tick per diagonal for small runs; a cancelled
    run holds the exact minimum over the completed diagonals; snapshots are monotone."""
    import oracle
    ts = mp.make_time_series([1, 2, 3, 4, 5, 6, 7, 8])
    ticks = []
    mp.aamp(ts, mp.ProfileConfig(3, mp.DistanceKind.euclidean()),
            lambda d, t: ticks.append((d, t)) or True)
    assert ticks and ticks[-1] == (5, 5) and len(ticks) == 5
    r = np.random.default_rng(506)
    t = r.uniform(-1, 1, 128)
    cfg = mp.ProfileConfig(8, mp.DistanceKind.euclidean())
    full = mp.aamp(mp.make_time_series(t), cfg)
    prev = None
    for stop in (1, 17, 60, 120):
        part = mp.aamp(mp.make_time_series(t), cfg, lambda d, tot, s=stop: d < s)
        assert np.all(part.distances >= full.distances - 1e-12)
        _, Pr, _ = oracle.scan(t, 8, k_lo=1, k_hi=stop + 1)
        assert np.all(np.abs(part.distances - Pr) <= 1e-9 * np.maximum(1, np.abs(Pr)))
        if prev is not None:
            assert np.all(part.distances <= prev + 1e-12)
        prev = part.distances
    assert np.array_equal(prev, full.distances)
