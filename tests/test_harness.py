"""QKVT container, RunConfig and the run / sweep / verify harness on the GPU path.

Fixtures under tests/golden/cli_* were produced by the REAL reference (oracle/make_cli_golden.py):
a container written by the reference's writer and the records its own CLI printed for it.  CPU
tests pin the reader, the config schema and the exit codes; GPU tests compare this harness's records
with the reference's (integers and densities exactly; float64 metrics to the tolerances stated)."""

import csv
import io
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import svgear_oracle as O
from paper_2603_08982_b200 import cli, config, tensorio

TENSOR = os.path.join(GOLDEN, "cli_blobs_d64.qkvt")
TENSOR_F64 = os.path.join(GOLDEN, "cli_blobs_d64_f64.qkvt")
CONFIG = os.path.join(GOLDEN, "cli_config.json")


def golden_records():
    with open(os.path.join(GOLDEN, "cli_run_records.jsonl"), encoding="utf-8") as fh:
        return [json.loads(line) for line in fh if line.strip()]


# ------------------------------------------------------------------------------------------------
# CPU: container, config, exit codes
# ------------------------------------------------------------------------------------------------
class TestTensorIO:
    def test_reads_what_the_reference_wrote(self):
        q, k, v = tensorio.read_tensor_file(TENSOR)
        want = [O.round_to_bf16(a) for a in O.blob_instance(384, 384, 64, 8, 12, 0.1, 11)]
        for got, ref in zip((q, k, v), want):
            assert got.dtype == np.float32 and got.shape == (384, 64)
            assert np.array_equal(got.astype(np.float64), ref)
        q64, k64, v64 = tensorio.read_tensor_file(TENSOR_F64)
        assert q64.dtype == np.float64 and np.array_equal(q64, want[0][:32]) and np.array_equal(v64, want[2][:32])

    @pytest.mark.parametrize("precision", ["double", "single"])
    def test_writer_is_byte_identical_to_the_reference(self, tmp_path, precision):
        src = TENSOR_F64 if precision == "double" else TENSOR
        q, k, v = tensorio.read_tensor_file(src)
        out = tmp_path / "copy.qkvt"
        tensorio.write_tensor_file(out, q, k, v, precision=precision)
        assert out.read_bytes() == open(src, "rb").read()

    def test_ragged_shapes_round_trip(self, tmp_path):
        rng = np.random.default_rng(0)
        q, k, v = rng.normal(size=(3, 5)), rng.normal(size=(7, 5)), rng.normal(size=(7, 2))
        p = tmp_path / "r.qkvt"
        tensorio.write_tensor_file(p, q, k, v)
        for got, ref in zip(tensorio.read_tensor_file(p), (q, k, v)):
            assert np.array_equal(got, ref)
        with pytest.raises(ValueError):
            tensorio.write_tensor_file(p, q[0], k, v)
        with pytest.raises(ValueError):
            tensorio.write_tensor_file(p, q, k, v, precision="half")

    def test_every_malformation_has_its_own_message(self, tmp_path):
        raw = bytearray(open(TENSOR_F64, "rb").read())

        def broken(edit):
            b = bytearray(raw)
            b = edit(b) or b
            p = tmp_path / "bad.qkvt"
            p.write_bytes(bytes(b))
            with pytest.raises(tensorio.TensorFormatError) as err:
                tensorio.read_tensor_file(p)
            return str(err.value)

        msgs = [
            broken(lambda b: b[:20]),
            broken(lambda b: b.__setitem__(slice(0, 4), b"QKVX")),
            broken(lambda b: b.__setitem__(4, 2)),
            broken(lambda b: b.__setitem__(6, 7)),
            broken(lambda b: b.__setitem__(7, 1)),
            broken(lambda b: b[:-8]),
            broken(lambda b: b + b"\0\0\0"),
        ]
        for m, word in zip(msgs, ("too short", "magic", "version", "dtype code", "reserved", "payload size", "trailing")):
            assert word in m, (word, m)
        assert len(set(msgs)) == len(msgs)


class TestRunConfig:
    def test_echo_matches_the_reference(self):
        for rec in golden_records():
            cfg = config.RunConfig.from_dict(rec["config"])
            assert cfg.to_dict() == rec["config"]
            assert list(cfg.to_dict()) == list(rec["config"])  # same key order in the JSON line

    @pytest.mark.parametrize("bad", [
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2},                                   # missing key
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "bogus": 1},              # unknown key
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 9, "cK": 2},                          # cQ > nQ
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "rho": 1.5},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "budgetMode": "perClusterTopP"},   # p missing
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "policy": "best"},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "seeds": []},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "seeds": [True]},
        {"nQ": 8.0, "nK": 8, "d": 4, "cQ": 2, "cK": 2},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "budgetMode": "perClusterTopP", "p": 0.5, "policy": "random"},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "precision": "half"},
        {"nQ": 8, "nK": 8, "d": 4, "cQ": 2, "cK": 2, "sigma": 0},
        [1, 2],
    ])
    def test_rejects(self, bad):
        with pytest.raises(config.ConfigError):
            config.RunConfig.from_dict(bad)

    def test_paper_preset(self):  # config.py:137-154
        cfg = config.apply_preset(config.RunConfig(n_q=1200, n_k=3600, d=64, c_q=5, c_k=5), "paper")
        assert (cfg.budget_mode, cfg.p, cfg.rho, cfg.c_q, cfg.c_k) == ("perClusterTopP", 0.85, None, 100, 1000)
        tiny = config.apply_preset(config.RunConfig(n_q=3, n_k=5, d=64, c_q=1, c_k=1), "paper")
        assert (tiny.c_q, tiny.c_k) == (3, 5)
        with pytest.raises(config.ConfigError):
            config.apply_preset(cfg, "fast")


class TestExitCodes:
    def test_config_errors_exit_2(self, tmp_path, capsys):
        bad = tmp_path / "bad.json"
        bad.write_text("{not json")
        assert cli.main(["run", TENSOR, "--config", str(bad)]) == 2
        bad.write_text(json.dumps({"nQ": 384, "nK": 384, "d": 64, "cQ": 8, "cK": 12, "zzz": 1}))
        assert cli.main(["run", TENSOR, "--config", str(bad)]) == 2
        assert cli.main(["sweep", TENSOR, "--config", CONFIG, "--density-grid", "0.1,x"]) == 2
        assert cli.main(["sweep", TENSOR, "--config", CONFIG, "--density-grid", "0.1,1.5"]) == 2
        assert cli.main(["sweep", TENSOR, "--config", CONFIG, "--density-grid", "0.1", "--policy", "nope"]) == 2
        assert "config error" in capsys.readouterr().err

    def test_input_errors_exit_3(self, tmp_path, capsys):
        junk = tmp_path / "junk.qkvt"
        junk.write_bytes(b"QKVT" + b"\0" * 10)
        assert cli.main(["run", str(junk), "--config", CONFIG]) == 3
        assert cli.main(["run", str(tmp_path / "missing.qkvt"), "--config", CONFIG]) == 3
        assert cli.main(["verify", TENSOR, "--config", str(tmp_path / "missing.json")]) == 3
        err = capsys.readouterr().err
        assert "input error" in err and "io error" in err

    def test_capability_errors_exit_4(self, tmp_path, capsys):
        assert cli.main(["run", TENSOR, "--config", CONFIG, "--policy", "oracleKnapsack"]) == 4
        small = tmp_path / "d16.qkvt"
        z = np.zeros((8, 16))
        tensorio.write_tensor_file(small, z, z, z)
        cfg = tmp_path / "c.json"
        cfg.write_text(json.dumps({"nQ": 8, "nK": 8, "d": 16, "cQ": 2, "cK": 2}))
        assert cli.main(["run", str(small), "--config", str(cfg)]) == 4
        assert "capability error" in capsys.readouterr().err

    @pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
    def test_no_cpu_path(self):
        assert cli.main(["run", TENSOR, "--config", CONFIG]) == 4


# ------------------------------------------------------------------------------------------------
# GPU: records against the reference CLI's
# ------------------------------------------------------------------------------------------------
def _close(a, b, rel):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


@pytest.mark.gpu
class TestRunAgainstReferenceRecords:
    @pytest.mark.parametrize("idx", range(7))
    def test_record(self, idx, tmp_path):
        ref = golden_records()[idx]
        cfg = tmp_path / "c.json"
        cfg.write_text(json.dumps(ref["config"]))
        for executor in ("fp32", "bf16"):
            out = tmp_path / f"{executor}.jsonl"
            rc = cli.main(["run", TENSOR, "--config", str(cfg), "--seed", str(ref["seed"]), "--no-timing",
                           "--executor", executor, "--out", str(out)])
            assert rc == 0
            lines = out.read_text().splitlines()
            assert len(lines) == 1
            got = json.loads(lines[0])
            assert "timing" not in got
            for key in ("policy", "density", "flopsTotal", "seed", "clusterCounts"):
                assert got[key] == ref[key], key
            assert got["config"] == dict(ref["config"], seeds=[ref["seed"]])
            assert _close(got["relaxedObjective"], ref["relaxedObjective"], 1e-5)
            assert _close(got["mapMse"], ref["mapMse"], 1e-5)
            if executor == "fp32":
                assert _close(got["outputMse"], ref["outputMse"], 1e-3)
            else:  # rounding an O(1) output to bf16 adds up to ~(2^-9)^2 of variance to the MSE
                assert 0.5 * ref["outputMse"] <= got["outputMse"] <= ref["outputMse"] + 2e-6

    def test_timing_field_and_stdout(self, capsys):
        assert cli.main(["run", TENSOR, "--config", CONFIG, "--seed", "0"]) == 0
        rec = json.loads(capsys.readouterr().out)
        assert rec["timing"]["seconds"] > 0 and rec["executor"] == "bf16"


@pytest.mark.gpu
class TestSweepAndVerify:
    def test_sweep_matches_the_reference_csv(self, tmp_path):
        out = tmp_path / "s.csv"
        rc = cli.main(["sweep", TENSOR, "--config", CONFIG, "--density-grid", "0.1,0.25,0.5", "--policy",
                       "topPCompensated,errorAwareCompensated", "--executor", "fp32", "--out", str(out)])
        assert rc == 0
        got = list(csv.reader(io.StringIO(out.read_text())))
        with open(os.path.join(GOLDEN, "cli_sweep.csv"), encoding="utf-8", newline="") as fh:
            ref = list(csv.reader(fh))
        assert got[0] == ref[0] == cli.CSV_HEADER.split(",")
        assert len(got) == len(ref) == 13
        for g, r in zip(got[1:], ref[1:]):
            assert g[0] == r[0] and float(g[1]) == float(r[1]) and g[5:] == r[5:], (g, r)
            assert _close(float(g[2]), float(r[2]), 1e-5)
            assert _close(float(g[3]), float(r[3]), 1e-5)
            assert _close(float(g[4]), float(r[4]), 1e-3)

    def test_default_policies_and_error_aware_wins_on_relaxed_objective(self, capsys):
        assert cli.main(["sweep", TENSOR, "--config", CONFIG, "--density-grid", "0.25", "--seed", "0"]) == 0
        rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))[1:]
        assert [r[0] for r in rows] == list(cli.SWEEP_DEFAULT_POLICIES)
        assert float(rows[1][2]) <= float(rows[0][2])

    @pytest.mark.parametrize("extra", [[], ["--preset", "paper"], ["--policy", "topPCompensated"]])
    def test_verify_passes(self, capsys, extra):
        rc = cli.main(["verify", TENSOR, "--config", CONFIG, *extra])
        report = json.loads(capsys.readouterr().out)
        assert rc == 0 and report["pass"] is True
        assert set(report["checks"]) == {"executorBf16VsFp32", "executorReference", "estimatorTensorVsFp32"}
        assert all(c["pass"] for c in report["checks"].values())
