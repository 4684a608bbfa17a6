"""Host-side checks of bench.py's driver contract (no GPU): the defaults, and the
reference arm's JSON line (the oracle timed on a bounded sample) on a small
stand-in for configs[3] so it runs in seconds here."""
import argparse
import json
import sys

import pytest

import bench
from paper_2210_07667_b200 import workloads as W


def test_defaults_meet_the_timing_rules(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.gpus == 1 and a.impl == "b200"
    assert a.warmup >= 3 and a.steps >= 1


@pytest.mark.parametrize("rank", [0, 1])
def test_reference_arm_line(monkeypatch, capsys, rank):
    small = W.config(3, small=True)
    monkeypatch.setattr(W, "config", lambda *a, **kw: small)
    monkeypatch.setenv("RANK", str(rank))
    monkeypatch.setenv("WORLD_SIZE", "2" if rank else "1")
    args = argparse.Namespace(gpus=2 if rank else 1, steps=2, warmup=1, impl="reference")
    bench.reference_arm(args)
    out = capsys.readouterr().out.strip()
    if rank:
        assert out == ""  # only rank 0 runs and prints the reference arm
        return
    line = json.loads(out.splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["value"] > 0 and line["ms_per_step"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == line["value"] and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["dtype"] == "f64" and line["data"] == "synthetic" and "workload" in line["config"]
