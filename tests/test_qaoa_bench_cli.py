"""qaoa-bench CLI on the B200 backend (paper_2407_13012_b200/cli.py, mirror of the
reference's cli.py): the record schema, file parsers and graph-suite writer on CPU;
the tasks, bench --jobs and kernel-bench on the GPU."""

import json

import pytest

import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import cli
from paper_2407_13012_b200.errors import ParseError

REFERENCE_KEYS = ["schema", "version", "task", "n", "p", "shots", "seed", "family", "backend", "timings", "result"]
DEVICE_KEYS = ["device", "gpus", "host_cores", "bytes_alg", "sweep_ms", "gbps", "roofline_frac"]


def test_record_schema_is_the_reference_schema_plus_device_fields():
    rec = cli.RunRecord("gradient", 20, 6, 1024, 1, "er50", "b200", timings={"precompute": 5, "gradient": 9},
                        result={"d_betas": [0.1]},
                        device={"device": {"name": "B200"}, "gpus": 1, "host_cores": 16, "bytes_alg": 1e9,
                                "sweep_ms": 1.0, "gbps": 1000.0, "roofline_frac": 0.15})
    row = rec.to_dict(True)
    assert row["schema"] == 1
    assert [k for k in row if k in REFERENCE_KEYS] == REFERENCE_KEYS  # same keys, same order
    assert all(k in row for k in DEVICE_KEYS)
    assert set(row["timings"]) == {"precompute", "gradient"}  # phases only, as in the reference
    bare = rec.to_dict(False)  # --no-timings: deterministic rows (no timings, no device rates)
    assert list(bare) == [k for k in REFERENCE_KEYS if k != "timings"]
    text = cli.render([rec], "jsonl", True)
    assert json.loads(text)["gbps"] == 1000.0
    head = cli.render([rec], "csv", True).splitlines()[0].split(",")
    assert "timings.precompute" in head and "device.name" in head and "result.d_betas" in head


def test_params_file(tmp_path):
    f = tmp_path / "p.txt"
    f.write_text("# depth\n2\n0.1 0.2\n0.3 0.4  # gammas\n")
    prm = cli.parse_params_file(f)
    assert prm.betas == (0.1, 0.2) and prm.gammas == (0.3, 0.4)
    f.write_text("3 ramp\n")
    assert cli.parse_params_file(f) == qs.linear_ramp_params(3)
    f.write_text("ramp\n")
    assert cli.parse_params_file(f, default_depth=2) == qs.linear_ramp_params(2)
    for bad in ("2\n0.1\n0.3 0.4\n", "x\n1\n1\n", "1\n1\n"):
        f.write_text(bad)
        with pytest.raises(ParseError):
            cli.parse_params_file(f)


def test_opt_config(tmp_path):
    f = tmp_path / "c.txt"
    f.write_text("max_iterations 7\ngrad_tol=1e-8 # tight\n")
    cfg = cli.read_opt_config(f)
    assert cfg.max_iterations == 7 and cfg.grad_tol == 1e-8
    f.write_text("bogus 1\n")
    with pytest.raises(ParseError):
        cli.read_opt_config(f)


def test_gen_graphs_and_usage_errors(tmp_path, capsys):
    assert cli.main(["gen-graphs", "--range", "6..7", "--instances", "2", "--out", str(tmp_path / "s")]) == 0
    files = sorted(p.name for p in (tmp_path / "s").glob("*.txt"))
    assert len(files) == 16 and "reg3_n06_i0.txt" in files  # 3 ER families x 2 n x 2, complete x 2, reg3 (even n) x 2
    g = qs.read_graph(tmp_path / "s" / "er50_n07_i1.txt")
    assert g.num_vertices == 7
    assert cli.main(["gen-graphs", "--range", "6-7", "--out", str(tmp_path / "t")]) == 1  # ParseError -> 1
    with pytest.raises(SystemExit) as e:  # argparse usage error -> 2
        cli.main(["expectation", "--graph", "x", "--backend", "accelerated"])
    assert e.value.code == 2
    assert cli.build_parser().parse_args(["kernel-bench", "-n", "16,20,24"]).n == "16,20,24"


@pytest.mark.gpu
def test_tasks_on_the_gpu(tmp_path, capsys):
    path = tmp_path / "k3.txt"
    qs.write_graph(path, qs.complete_graph(3))
    zero = tmp_path / "zero.txt"
    zero.write_text("1\n0\n0\n")
    assert cli.main(["expectation", "--graph", str(path), "-p", "1", "--params", str(zero), "--no-timings"]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["backend"] == "b200" and rec["result"]["value"] == pytest.approx(-1.5, abs=1e-12)
    g20 = tmp_path / "g20.txt"
    qs.write_graph(g20, qs.erdos_renyi(20, 0.5, seed=3))
    assert cli.main(["gradient", "--graph", str(g20), "-p", "3", "--backend", "gpu"]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["result"]["layer_applications"] == 19
    assert rec["bytes_alg"] > 0 and 0 < rec["roofline_frac"] < 1.5 and rec["gpus"] == 1
    assert cli.main(["sample", "--graph", str(g20), "-p", "2", "--shots", "500", "--seed", "4"]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert len(rec["result"]["records"]) == 500
    assert cli.main(["optimize", "--graph", str(path), "-p", "2", "--no-timings"]) == 0
    assert json.loads(capsys.readouterr().out)["result"]["value"] == pytest.approx(-2.0, abs=1e-6)
    suite = tmp_path / "suite"
    assert cli.main(["gen-graphs", "--range", "6..13", "--instances", "1", "--families", "er50,reg3",
                     "--out", str(suite)]) == 0
    capsys.readouterr()
    out = tmp_path / "bench.jsonl"
    assert cli.main(["bench", "--suite", str(suite), "--task", "gradient", "--jobs", "4", "--out", str(out)]) == 0
    rows = [json.loads(x) for x in out.read_text().splitlines()]
    assert len(rows) == 8 + 4 and all(r["task"] == "gradient" for r in rows)
    assert cli.main(["kernel-bench", "-n", "14,16", "-p", "2", "--repeats", "2", "--json"]) == 0
    lines = [json.loads(x) for x in capsys.readouterr().out.splitlines() if x.startswith("{")]
    assert [x["n"] for x in lines] == [14, 16] and lines[1]["phases"]["gradient"]["ms"] > 0
