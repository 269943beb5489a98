"""CLI reports are byte-identical to the reference's (tests/golden/cli.json).

`map` runs K1/K2 on the GPU (marked gpu); the analytic reports run anywhere.
"""

import contextlib
import io

import pytest

from conftest import golden
from paper_2507_17087_b200.cli import main
from paper_2507_17087_b200.sweep import TABLE3_AREAS, TABLE3_GPUS, TABLE3_RATIOS, sweep_configs, sweep_groups


def _run(case, tmp_path):
    argv = [case["cmd"]]
    path = None
    if case["mapper"]:
        path = tmp_path / "m.mapper"
        path.write_text(case["source"])
        argv.append(str(path))
    argv += case["args"]
    buf, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
        code = main(argv)
    text = buf.getvalue()
    if path:
        text = text.replace(str(path), "@MAPPER@")
    return code, text


CASES = golden("cli")


@pytest.mark.parametrize("case", [c for c in CASES if c["cmd"] != "map"],
                         ids=lambda c: f"{c['cmd']}-{'-'.join(c['args'][:3])}")
def test_host_reports_match_reference(case, tmp_path):
    code, text = _run(case, tmp_path)
    assert code == case["exit"]
    assert text == case["stdout"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["cmd"] == "map"],
                         ids=lambda c: f"map-{c['mapper']}-{c['args'][1]}")
def test_map_report_matches_reference(case, tmp_path):
    code, text = _run(case, tmp_path)
    assert code == case["exit"]
    assert text == case["stdout"]


def test_sweep_directional():
    recs = sweep_configs(TABLE3_RATIOS, TABLE3_AREAS, TABLE3_GPUS, 4)
    assert len(recs) == 180
    assert all(r["improvement_pct"] >= 0 for r in recs)
    g = {(x["parameter"], str(x["value"])): x["geomean_improvement_pct"] for x in sweep_groups(recs)}
    assert g[("aspect_ratio", "1:32")] > g[("aspect_ratio", "1:1")]
