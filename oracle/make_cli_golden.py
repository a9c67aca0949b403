"""Generate the harness fixtures by running the REAL reference CLI.

Build container only (needs /root/reference):

    python oracle/make_cli_golden.py

Writes under tests/golden/:
  cli_blobs_d64.qkvt   a QKVT container WRITTEN BY THE REFERENCE (`tensorio.write_tensor_file`,
                       single precision; the values are bf16-representable, so float32 is exact)
  cli_blobs_d64_f64.qkvt  the first 32 rows of each matrix in double precision (reader test)
  cli_config.json      the RunConfig the records below were produced with
  cli_run_records.jsonl   `routedattn run --no-timing` output for the policies / budget modes the
                       GPU harness supports (seeds 0 and 1)
  cli_sweep.csv        `routedattn sweep` over topPCompensated,errorAwareCompensated x 3 densities
"""

from __future__ import annotations

import io
import json
import os
import sys
from contextlib import redirect_stdout

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from routedattn import cli, tensorio  # noqa: E402  (the reference)

from oracle import svgear_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
N, D, CQ, CK = 384, 64, 8, 12


def run_cli(argv):
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == 0, (argv, rc)
    return buf.getvalue()


def main():
    q, k, v = (O.round_to_bf16(a) for a in O.blob_instance(N, N, D, CQ, CK, 0.1, 11))
    tensor = os.path.join(OUT, "cli_blobs_d64.qkvt")
    tensorio.write_tensor_file(tensor, q, k, v, precision="single")
    tensorio.write_tensor_file(os.path.join(OUT, "cli_blobs_d64_f64.qkvt"), q[:32], k[:32], v[:32],
                               precision="double")
    base = {"nQ": N, "nK": N, "d": D, "cQ": CQ, "cK": CK, "rho": 0.25, "seeds": [0, 1]}
    cfg = os.path.join(OUT, "cli_config.json")
    with open(cfg, "w", encoding="utf-8") as fh:
        json.dump(base, fh, indent=1, sort_keys=True)
        fh.write("\n")
    top_p = dict(base, budgetMode="perClusterTopP", p=0.85, rho=None)
    cfg_p = "/tmp/cli_config_top_p.json"
    with open(cfg_p, "w", encoding="utf-8") as fh:
        json.dump(top_p, fh)
    plain = dict(base, estimatorMode="plain")
    cfg_plain = "/tmp/cli_config_plain.json"
    with open(cfg_plain, "w", encoding="utf-8") as fh:
        json.dump(plain, fh)
    lines = ""
    lines += run_cli(["run", tensor, "--config", cfg, "--no-timing"])
    lines += run_cli(["run", tensor, "--config", cfg, "--no-timing", "--policy", "topPCompensated"])
    lines += run_cli(["run", tensor, "--config", cfg_p, "--no-timing"])
    lines += run_cli(["run", tensor, "--config", cfg_plain, "--no-timing", "--seed", "0"])
    with open(os.path.join(OUT, "cli_run_records.jsonl"), "w", encoding="utf-8") as fh:
        fh.write(lines)
    csv_text = run_cli(["sweep", tensor, "--config", cfg, "--density-grid", "0.1,0.25,0.5",
                        "--policy", "topPCompensated,errorAwareCompensated", "--workers", "1"])
    with open(os.path.join(OUT, "cli_sweep.csv"), "w", encoding="utf-8", newline="") as fh:
        fh.write(csv_text)
    print(lines)
    print(csv_text)


if __name__ == "__main__":
    main()
