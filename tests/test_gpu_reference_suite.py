"""The reference's own hot-path test files, unchanged, against the drop-in.

`pwadvect` is resolved to this package through tests/dropin_alias (the hot-
path modules grid / kernel / schedules are ours and run on the GPU; the
out-of-scope FPGA modelling modules are the stock files), and the stock test
files installed with the reference in baseline/_ref/tests run in a
subprocess with pytest:

* test_kernel.py      (pkg/tests/test_kernel.py:32-192: goldens, naive oracle,
                       symmetry, closed forms, point ops, equivariance)
* test_grid.py        (pkg/tests/test_grid.py:24-127: layout, LCG, fill, wrap,
                       field files, digests)
* test_schedules.py   (pkg/tests/test_schedules.py:63-188: variants, engines,
                       traffic closed forms, comparator)
* test_acceptance.py  criteria 7-9 (pkg/tests/test_acceptance.py:116-192)
* test_cli.py         the `bench` command's tests (pkg/tests/test_cli.py:35-79):
                       the stock CLI (cli.py:120-163), unmodified, calling OUR
                       run_schedule per variant — checksums, traffic columns,
                       determinism of the report rows

and the reference's demos that call the hot path (the callers SURVEY.md §8b
lists), unchanged: demos/01_stencil_basics.py and 02_schedule_traffic.py run
once against the drop-in and once against the stock package; their outputs
(checksums, identities, traffic counters) must be identical line for line
apart from the wall-time column.

No test is skipped or expected to fail. baseline/_ref is not in git (the
reference is installed there once); without it this file skips.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
STOCK_TESTS = ROOT / "baseline" / "_ref" / "tests"
STOCK_DEMOS = ROOT / "baseline" / "_ref" / "demos"
ALIAS = ROOT / "tests" / "dropin_alias"

FILES = {
    "test_kernel.py": None,
    "test_grid.py": None,
    "test_schedules.py": None,
    "test_acceptance.py": "criterion_7 or criterion_8 or criterion_9",
    "test_cli.py": "bench",
}


def _run(name, select):
    if not (STOCK_TESTS / name).exists():
        pytest.skip("stock reference tests not installed in baseline/_ref")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ALIAS), str(ROOT)] + ([env["PYTHONPATH"]]
                                                                   if env.get("PYTHONPATH") else []))
    cmd = [sys.executable, "-m", "pytest", "-q", "-s", "-p", "no:cacheprovider",
           "--rootdir", str(STOCK_TESTS), str(STOCK_TESTS / name)]
    if select:
        cmd += ["-k", select]
    # the alias must win over any installed pwadvect: check before trusting the run
    probe = subprocess.run([sys.executable, "-c", "import pwadvect, pwadvect.kernel as k; "
                            "print(k.run_reference.__module__)"], env=env, capture_output=True,
                           text=True, cwd=STOCK_TESTS)
    assert probe.returncode == 0, probe.stderr
    assert probe.stdout.strip() == "paper_2010_01545_b200.stencil", probe.stdout
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=STOCK_TESTS, timeout=1800)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and "skipped" not in res.stdout and "xfail" not in res.stdout, tail
    return res.stdout


@pytest.mark.parametrize("name", sorted(FILES))
def test_reference_test_file_unchanged(name):
    out = _run(name, FILES[name])
    if name == "test_acceptance.py":
        for n in (7, 8, 9):
            assert f"ACCEPTANCE PASS  {n}" in out, out[-2000:]


def _demo_output(path, pythonpath):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(str(p) for p in pythonpath)
    res = subprocess.run([sys.executable, str(path)], env=env, capture_output=True, text=True,
                         cwd=path.parent, timeout=900)
    assert res.returncode == 0, (res.stdout + res.stderr)[-3000:]
    return res.stdout


def _without_wall(line: str) -> str:
    """demo 02's table rows end in a wall-time column (schedules.py:220-228)."""
    head = line.split(" ", 1)[0]
    if head in ("reference", "column_buffered", "y_batched", "x_reordered"):
        return line.rsplit(None, 1)[0]
    return line


@pytest.mark.parametrize("demo", ["01_stencil_basics.py", "02_schedule_traffic.py"])
def test_reference_demo_unchanged(demo):
    path = STOCK_DEMOS / demo
    if not path.exists():
        pytest.skip("stock reference demos not installed in baseline/_ref")
    ours = _demo_output(path, [ALIAS, ROOT])
    stock = _demo_output(path, [ROOT / "baseline" / "_ref"])
    a = [_without_wall(x) for x in ours.splitlines()]
    b = [_without_wall(x) for x in stock.splitlines()]
    assert a == b, "\n".join(f"{x!r} | {y!r}" for x, y in zip(a, b) if x != y)
    assert "checksum" in ours


def test_whole_reference_suite_unchanged():
    """Every stock test file in one run (the FPGA modelling tests included:
    those modules are the stock files, but their grids, fields and any
    stencil they evaluate come from the drop-in): nothing may fail or skip."""
    if not STOCK_TESTS.exists():
        pytest.skip("stock reference tests not installed in baseline/_ref")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ALIAS), str(ROOT)])
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          "--rootdir", str(STOCK_TESTS), str(STOCK_TESTS)], env=env,
                         capture_output=True, text=True, cwd=STOCK_TESTS, timeout=1800)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    last = res.stdout.strip().splitlines()[-1]
    n = int(last.split(" passed")[0].split()[-1])
    n_stock = sum(line.lstrip().startswith("def test_") for f in STOCK_TESTS.glob("test_*.py")
                  for line in f.read_text().splitlines())
    assert n >= n_stock and "skipped" not in last and "failed" not in last, last
