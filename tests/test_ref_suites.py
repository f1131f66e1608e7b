"""The reference's own unit suites (proj/tests/test_{core,advantage,optim,policy,envsim,
placement}.cpp), compiled in place against the unmodified reference objects that oracle/_ref
is built from (oracle/Makefile `suites`, doctest replaced by oracle/doctest_shim/doctest.h since
doctest is not vendored), must pass: the checker the parity tests pin against is the reference
as its authors test it. Skipped where /root/reference is absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle")
SUITES = ["test_core", "test_advantage", "test_optim", "test_policy", "test_envsim", "test_placement"]

pytestmark = pytest.mark.skipif(not os.path.isdir("/root/reference/proj/tests"),
                                reason="/root/reference not present")


@pytest.fixture(scope="module")
def built():
    subprocess.run(["make", "-s", "-j8", "-C", ORACLE, "suites"], check=True, capture_output=True)
    return os.path.join(ORACLE, "_ref", "suites")


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(built, suite, tmp_path):
    r = subprocess.run([os.path.join(built, suite)], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    summary = r.stdout.strip().splitlines()[-1]
    assert r.returncode == 0, r.stdout[-2000:]
    assert "| 0 failed | assertions:" in summary and summary.endswith("| 0 failed"), summary


def test_shim_counts_subcases_and_failures(tmp_path):
    """The shim runs each flat SUBCASE exactly once per test case and reports failures."""
    src = tmp_path / "t.cpp"
    src.write_text('''
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
#include <stdexcept>
static int a = 0, b = 0, c = 0;
TEST_CASE("subcases") {
  ++c;
  SUBCASE("a") { ++a; CHECK(1.0 == doctest::Approx(1.0 + 1e-9)); }
  SUBCASE("b") { ++b; CHECK_THROWS_AS(throw std::runtime_error("x"), std::runtime_error); }
}
TEST_CASE("counts") { CHECK(a == 1); CHECK(b == 1); CHECK(c == 2); }
TEST_CASE("fails") { CHECK(2 + 2 == 5); CHECK_FALSE(true); CHECK(0.1 == doctest::Approx(0.2)); }
''')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ORACLE, "doctest_shim"), str(src), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1
    assert "test cases: 3 | 1 failed | assertions: 8 | 3 failed" in r.stdout, r.stdout


def test_reference_acceptance_criteria_pass(tmp_path):
    """proj/tests/acceptance.cpp — the reference's nine acceptance criteria (GAE vs the
    double-sum oracle, FD gradients, granularity identity, GRPO standardization / exhaustive
    filter, partial reset, scheduling invariance across placements / k / backends, virtual-clock
    throughput band, ToyReach learning, chunk_step equivalence) built in place with its harness
    (oracle/Makefile `acceptance`)."""
    subprocess.run(["make", "-s", "-j8", "-C", ORACLE, "acceptance"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(ORACLE, "_ref", "suites", "acceptance")], cwd=tmp_path,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "all 9 acceptance criteria passed" in r.stdout, r.stdout[-3000:]
