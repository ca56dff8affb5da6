"""The C++ drop-in (include/vpipe/vocab_math.hpp): the restated reference
unit tests and the `verify` CLI contract of P/tests/cli_test.sh:32-35."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOLS = os.path.join(ROOT, "tools")


def _build():
    subprocess.run(["make", "-s", "-C", TOOLS, "vpipe_verify", "test_vocab_math_gpu"], check=True)


def _verify(*args):
    return subprocess.run([os.path.join(TOOLS, "vpipe_verify"), *args], capture_output=True, text=True, timeout=600)


def test_verify_usage_errors_exit_2():
    _build()
    r = _verify("--bogus", "1")
    assert r.returncode == 2 and "unknown option" in r.stderr
    r = _verify("--devices")
    assert r.returncode == 2


@pytest.mark.gpu
def test_cpp_unit_tests_restated_from_the_reference():
    _build()
    r = subprocess.run([os.path.join(TOOLS, "test_vocab_math_gpu")], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


@pytest.mark.gpu
def test_verify_cli_contract():
    # cli_test.sh:32-35: verify passes; p=1 passes; --fault-scale 1.01 exits 1 naming alg1
    _build()
    r = _verify("--seed", "0")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 5  # device oracle, naive, alg1, alg2 vs the CPU oracle + input layer
    r = _verify("--devices", "1")
    assert r.returncode == 0, r.stdout + r.stderr
    r = _verify("--fault-scale", "1.01")
    assert r.returncode == 1
    assert any(line.startswith("alg1") and line.endswith("FAIL") for line in r.stdout.splitlines())
    r = _verify("--devices", "5", "--vocab", "32")  # pad_vocab_size makes V=40, divisible by 5
    assert r.returncode == 0, r.stdout + r.stderr
    r = _verify("--hidden", "4096", "--vocab", "128256", "--devices", "8", "--batch", "1", "--seq-len", "16")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_verify_detects_a_corrupted_logits_kernel():
    # a fault common to every p (K1 logits scaled by 1 + 2e-3) must fail
    # against the independent CPU oracle
    _build()
    r = _verify("--inject-k1-fault", "2000", "--hidden", "64", "--vocab", "256")
    assert r.returncode == 1, r.stdout + r.stderr
    assert any(line.startswith("alg2") and line.endswith("FAIL") for line in r.stdout.splitlines())
    assert any(line.startswith("device_oracle") and line.endswith("FAIL") for line in r.stdout.splitlines())


@pytest.mark.gpu
def test_verify_with_ranks_through_the_loopback_backend():
    _build()
    for p in ("2", "4"):
        r = _verify("--placement", "loopback", "--devices", p, "--hidden", "64", "--vocab", "512")
        assert r.returncode == 0, r.stdout + r.stderr
