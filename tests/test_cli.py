"""CLI parity with the reference's `ntpsim shardmap` / `verify` (cli.py:328-382,
tests/test_cli.py:21-71): same strings, JSON shapes and exit codes."""

import json
import subprocess
import sys

import pytest
import torch

from paper_2504_06095_b200.cli import main

from conftest import ROOT


def run_cli(capsys, *argv):
    rc = main(list(argv))
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_shardmap_prints_contrast_stats(capsys):
    rc, out, _ = run_cli(capsys, "shardmap", "--k", "12000", "--n1", "32", "--n2", "30")
    assert rc == 0
    assert "max 25 sent / 375 received" in out
    assert "750 columns" in out
    assert out.splitlines()[0] == "shard map: k=12000 n1=32 n2=30"
    assert "  comp shards per rank: 375..375" in out
    assert "  sync shards per rank: 400..400 on 30 ranks" in out


def test_shardmap_equal_groups_has_empty_plans(capsys):
    rc, out, _ = run_cli(capsys, "shardmap", "--k", "8", "--n1", "4", "--n2", "4")
    assert rc == 0 and "0 columns over 0 links" in out


def test_shardmap_json_shape(capsys):
    rc, out, _ = run_cli(capsys, "shardmap", "--k", "100", "--n1", "8", "--n2", "6", "--json")
    assert rc == 0
    doc = json.loads(out)
    assert set(doc) == {"map", "pre_sync", "post_sync"}
    assert doc["map"]["k"] == 100
    assert set(doc["pre_sync"]) == {"direction", "total_cols_moved", "max_cols_sent",
                                    "max_cols_received", "links"}
    assert doc["post_sync"]["total_cols_moved"] == doc["pre_sync"]["total_cols_moved"]


def test_shardmap_rejects_invalid_groups(capsys):
    rc, _, err = run_cli(capsys, "shardmap", "--k", "8", "--n1", "4", "--n2", "6")
    assert rc == 2
    assert err.strip() == "error: reduced degree n2=6 exceeds healthy degree n1=4"


def test_verify_shard_invariants(capsys):
    rc, out, _ = run_cli(capsys, "verify", "--suite", "shard-invariants")
    assert rc == 0 and out.startswith("PASS shard-invariants")


def test_verify_json(capsys):
    rc, out, _ = run_cli(capsys, "verify", "--suite", "shard-invariants", "--json")
    doc = json.loads(out)
    assert rc == 0 and doc["passed"] and doc["suites"][0]["name"] == "shard-invariants"


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_2504_06095_b200.cli", "--version"],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0 and "ntp-b200" in r.stdout


@pytest.mark.gpu
def test_verify_tp_numerics_on_device(capsys):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rc, out, _ = run_cli(capsys, "verify", "--suite", "tp-numerics")
    assert rc == 0, out
    assert out.startswith("PASS tp-numerics")


@pytest.mark.gpu
def test_verify_all_four_suites(capsys):
    """`verify` with no suite runs the reference's four suites (cli.py:320-325)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rc, out, _ = run_cli(capsys, "verify")
    assert rc == 0, out
    assert [l.split(":")[0] for l in out.splitlines() if l.startswith("PASS")] == [
        "PASS shard-invariants", "PASS tp-numerics", "PASS grad-finite-diff", "PASS golden"]
    assert not any(l.startswith("FAIL") for l in out.splitlines())


@pytest.mark.gpu
def test_verify_golden_json(capsys):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rc, out, _ = run_cli(capsys, "verify", "--suite", "golden", "--json")
    doc = json.loads(out)
    assert rc == 0 and doc["passed"] is True and doc["suites"][0]["name"] == "golden"


@pytest.mark.gpu
def test_verify_golden_catches_activation_drift(capsys, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2504_06095_b200.tpnumerics as tpn
    monkeypatch.setattr(tpn, "GELU_C", 0.0447)
    rc, out, _ = run_cli(capsys, "verify", "--suite", "golden")
    assert rc == 1 and "FAIL golden" in out and "case:" in out


def test_golden_fixture_shipped_with_package():
    """The package carries the reference's golden fixture (verify --suite golden)."""
    from paper_2504_06095_b200.cli import _golden_fixture
    with open(f"{ROOT}/tests/golden/golden_mlp.json") as f:
        assert _golden_fixture() == json.load(f)


def test_verify_suite_names():
    from paper_2504_06095_b200.cli import SUITES
    assert list(SUITES) == ["shard-invariants", "tp-numerics", "grad-finite-diff", "golden"]
