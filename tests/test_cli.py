"""CLI front end (cli.py; REF cli.py): argument parsing, exit codes, and the
reference's per-iteration ``report`` series from a trace in the reference
schema (CPU); the decode -> report round trip on a GPU."""
import csv
import json

import pytest

from paper_2605_02189_b200 import cli
from paper_2605_02189_b200.trace import EventTrace


def test_report_series_from_trace(tmp_path):
    tr = EventTrace()
    for it in range(3):
        tr.emit(0.01 * it, "stage_compute_start", phase="decode", stage=0, iter=it, batch=it % 2,
                exec_seconds=0.005 + 0.001 * it, capacity_tokens=1000, next_residual_tokens=100 * it,
                next_prefetched_tokens=10 * it)
        tr.emit(0.01 * it, "stage_compute_start", phase="decode", stage=1, iter=it, batch=it % 2)
        tr.emit(0.01 * it + 0.005, "stage_compute_end", phase="decode", stage=0, iter=it, batch=it % 2)
    tr.finalize()
    path = tmp_path / "t.jsonl"
    tr.to_jsonl(str(path))
    out = tmp_path / "r.csv"
    assert cli.main(["report", "--trace", str(path), "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["iter", "exec_seconds", "resident_fraction", "prefetched_fraction"]
    assert [r[0] for r in rows[1:]] == ["0", "1", "2"]
    assert float(rows[3][2]) == pytest.approx(0.2) and float(rows[3][3]) == pytest.approx(0.02)


def test_exit_codes(tmp_path):
    assert cli.main(["report", "--trace", str(tmp_path / "missing.jsonl")]) == 2
    bad = tmp_path / "bad.jsonl"
    bad.write_text("{not json\n")
    assert cli.main(["report", "--trace", str(bad)]) == 2
    assert cli.main(["decode", "--model", "no-such-model"]) == 2


@pytest.mark.gpu
def test_decode_then_report(tmp_path):
    tr, met, rep = tmp_path / "t.jsonl", tmp_path / "m.json", tmp_path / "r.csv"
    assert cli.main(["decode", "--requests", "16", "--prompt", "40", "--gen", "8", "--micro-batches", "4",
                     "--horizon", "12", "--prefill", "--trace", str(tr), "--metrics", str(met)]) == 0
    record = json.load(open(met))
    assert record["iterations"] == 12 and record["tokens_per_second"] > 0
    kinds = {json.loads(line)["kind"] for line in open(tr)}
    assert {"stage_compute_start", "stage_compute_end", "transfer_start", "transfer_end"} <= kinds
    assert cli.main(["report", "--trace", str(tr), "--out", str(rep)]) == 0
    assert len(list(csv.reader(open(rep)))) == 13


@pytest.mark.gpu
def test_compare_policies(tmp_path):
    out = tmp_path / "c.csv"
    assert cli.main(["compare", "--requests", "24", "--prompt", "40", "--gen", "8", "--host-tokens", "700",
                     "--policies", "dynamic,no_prefetch", "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0][0] == "policy" and [r[0] for r in rows[1:]] == ["dynamic", "no_prefetch"]
    assert all(float(r[1]) > 0 for r in rows[1:])
