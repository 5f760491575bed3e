"""CLI and plain-C client: input errors are rejected on any host (exit 1); on the GPU box the
CLI and the C example both recover C1's planted factor."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_1310_3809_b200", *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_cli_input_errors():
    assert _cli("factor", "--n", "xyz").returncode == 1
    assert _cli("factor", "--n", "10").returncode == 1          # even
    assert _cli("factor", "--n", "f" * 130).returncode == 1     # 520 bits > 510
    assert _cli("factor", "--n", "8f", "--family", "small", "--schedule", "primes").returncode == 1
    assert _cli("factor", "--n", "8f", "--b1", "1").returncode == 1


def _build_c_example():
    exe = os.path.join(ROOT, "examples", "ecm_factor")
    lib = os.path.join(ROOT, "paper_1310_3809_b200")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "ecm_factor.c"),
                    "-L", lib, "-lecmgpu", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_c_example_compiles_and_rejects_bad_input():
    exe = _build_c_example()
    assert subprocess.run([exe, "zz"], capture_output=True).returncode == 1


@pytest.mark.gpu
def test_cli_and_c_example_find_planted_factor():
    from workload import ecm_config
    cfg = ecm_config("C1")
    r = _cli("factor", "--n", f"{cfg['N']:x}", "--b1", "2000", "--curves", "256", "--seed", "1")
    assert r.returncode == 0, r.stderr
    assert str(cfg["p"]) in r.stdout
    r = _cli("factor", "--n", f"{cfg['N']:x}", "--b1", "2000", "--curves", "256", "--schedule", "primes")
    assert r.returncode == 0 and str(cfg["p"]) in r.stdout
    r = _cli("factor", "--n", f"{cfg['N']:x}", "--b1", "2000", "--curves", "256", "--family", "small")
    assert r.returncode == 0 and str(cfg["p"]) in r.stdout
    exe = _build_c_example()
    out = subprocess.run([exe, f"{cfg['N']:x}", "2000", "256", "7"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert f"factor 0x{cfg['p']:x}" in out.stdout
