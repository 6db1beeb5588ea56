"""CLI parity with the reference's QR subcommands (golden outputs captured
from the reference CLI) and the C ABI surface of libtqr.so."""
import ctypes as C
import os
import re

import pytest

from paper_1303_3182_b200 import _lib
from paper_1303_3182_b200.cli import main

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("argv", [
    "qr-coarse --p 15 --q 6 --algo greedy --check",
    "qr-coarse --p 9 --q 4 --algo fibonacci",
    "qr-tiled --p 15 --q 6 --algo greedy --check",
    "qr-tiled --p 15 --q 6 --algo plasmatree --bs 5",
    "qr-tiled --p 10 --q 4 --algo grasap",
    "qr-tiled --p 8 --q 4 --algo flattree --family TS",
    "qr-coarse --p 3 --q 5",
])
def test_cli_matches_reference(golden, capsys, argv):
    rec = golden["cli"][argv]
    rc = main(argv.split())
    cap = capsys.readouterr()
    assert rc == rec["rc"]
    assert cap.out == rec["out"]
    assert cap.err == rec["err"]


def test_cli_flags_and_outdir(tmp_path, monkeypatch, capsys):
    assert main(["qr-tiled", "--p", "15"]) == 2
    assert main(["nonsense"]) == 2
    monkeypatch.setenv("TILEDAG_OUTDIR", str(tmp_path))
    assert main(["qr-coarse", "--p", "6", "--q", "3", "--list", "--out", "t"]) == 0
    assert (tmp_path / "t").read_text().startswith("i\\k,1,2,3")
    assert (tmp_path / "t.elim").read_text().startswith("k,i,piv,step")
    capsys.readouterr()
    _, o1 = main(["qr-tiled", "--p", "10", "--q", "4", "--algo", "grasap"]), capsys.readouterr().out
    _, o2 = main(["qr-tiled", "--p", "10", "--q", "4", "--algo", "grasap"]), capsys.readouterr().out
    assert o1 == o2


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "tqr.h")).read()
    decl = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(tqr_\w+)\s*\(", hdr, re.M))
    assert len(decl) >= 25
    L = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(decl) if not hasattr(L, s)]
    assert not missing, missing
    assert set(decl) == set(_lib.SIGNATURES), set(decl) ^ set(_lib.SIGNATURES)
    assert _lib.lib().tqr_abi_version() == 1


def test_error_status_mapping():
    lib = _lib.lib()
    n = C.c_int64()
    x = C.c_int32()
    rc = lib.tqr_coarse_schedule(3, 5, b"greedy", None, None, 0, C.byref(n), C.byref(x))
    assert rc == _lib.TQR_EVALUE and lib.tqr_last_error() == b"need p >= q >= 1"
    with pytest.raises(ValueError, match="unknown coarse algorithm 'bogus'"):
        _lib.check(lib.tqr_coarse_schedule(4, 3, b"bogus", None, None, 0, C.byref(n), C.byref(x)))


@pytest.mark.parametrize("cmd,kind,key", [("qr-coarse --p 15 --q 6 --algo fibonacci --check", "coarse", "fibonacci"),
                                          ("qr-tiled --p 15 --q 6 --algo plasmatree --bs 5 --check", "tiled",
                                           "plasmatree/5"),
                                          ("qr-tiled --p 15 --q 6 --algo binarytree --check", "tiled",
                                           "binarytree")])
def test_cli_check_compares_every_cell(monkeypatch, capsys, cmd, kind, key):
    """--check compares all 15x6 cells (reference cli.py:119-127, :141-148):
    every table passes as built, and a corrupted cell in an inner row is
    reported by its (i,k) with exit code 1."""
    from paper_1303_3182_b200 import cli
    assert main(cmd.split()) == 0
    capsys.readouterr()
    good = cli._golden_cells(kind, key)
    assert len(good) == sum(min(i - 1, 6) for i in range(2, 16))
    bad = dict(good)
    bad[(4, 2)] += 1
    monkeypatch.setattr(cli, "_golden_cells", lambda k, kk: bad)
    assert main(cmd.split()) == 1
    assert "(4,2)" in capsys.readouterr().err


def _build_c_example(tmp_path):
    """Compile tests/c_host/example.c (a plain C host of include/tqr.h) with
    gcc against the in-tree libtqr.so; None if no C compiler."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        return None
    lib_dir = os.path.join(ROOT, "paper_1303_3182_b200")
    exe = str(tmp_path / "tqr_example")
    cmd = [cc, "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c_host", "example.c"), "-L", lib_dir, "-ltqr",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_host_schedule(tmp_path):
    """The C ABI from a C program (no Python): build_tree golden cp/weight and
    the reference's error message, without a GPU."""
    import subprocess
    exe = _build_c_example(tmp_path)
    if exe is None:
        pytest.skip("no C compiler")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cp 78, total weight 640" in r.stdout and "need p >= q >= 1" in r.stdout
