"""CLI harness: parsing, precedence, validation exit codes (CPU) and the
output formats on the GPU (reference tests/test_cli.py)."""

import json

import numpy as np
import pytest

from paper_2309_10477_b200 import cli
from paper_2309_10477_b200.cli import CSV_HEADER, main, parse_config

FAST = ["--paths", "4096", "--runs", "2", "--steps", "16", "--scheme", "milstein"]


def run(capsys, argv):
    code = main(argv)
    cap = capsys.readouterr()
    return code, cap.out, cap.err


class TestParsing:
    def test_defaults(self):
        _, man, _ = parse_config(["price"])
        p = man.params
        assert (p.kappa, p.theta, p.sigma, p.v0, p.r) == (6.21, 0.019, 0.61, 0.010201, 0.0319)
        assert man.spec.strike == man.spec.spot == 100.0 and man.spec.maturity == 1.0
        assert man.config.scheme == "exact" and man.config.precision == "fp32"  # reference default

    def test_sobol_bridge_flag_and_file(self, tmp_path):
        _, man, _ = parse_config(["greeks", "--scheme", "milstein", "--sampler", "sobol",
                                  "--sobol-highdim-ack", "--sobol-bridge", "8"])
        assert man.config.sobol_bridge == 8
        f = tmp_path / "c.cfg"
        f.write_text("scheme = milstein\nsampler = sobol\nsobol_highdim_ack = yes\nsobol_bridge = 4\n")
        _, man, _ = parse_config(["greeks", "--config", str(f)])
        assert man.config.sobol_bridge == 4

    def test_asian_dates(self):
        _, man, _ = parse_config(["price", "--product", "asian", "--averaging-times",
                                  "0.25,0.5,0.75,1"])
        assert man.spec.averaging_times == (0.25, 0.5, 0.75, 1.0)

    def test_flag_beats_file_beats_default(self, tmp_path):
        f = tmp_path / "cfg.txt"
        f.write_text("paths = 512\nseed = 9  # comment\nprecision = fp64\nsobol_scramble = yes\n")
        _, man, _ = parse_config(["price", "--config", str(f), "--paths", "128"])
        assert man.config.n_paths == 128 and man.config.seed == 9
        assert man.config.precision == "fp64" and man.config.sobol_scramble is True

    def test_bench_sweep_grid(self):
        _, man, merged = parse_config(["bench", "--scheme", "euler,milstein", "--paths", "100,200",
                                       "--steps", "8"])
        assert merged["_sweep"] == [("euler", 100, 8), ("euler", 200, 8), ("milstein", 100, 8),
                                    ("milstein", 200, 8)]
        assert man.config.scheme == "euler"

    def test_manifest_flat(self):
        _, man, _ = parse_config(["greeks", "--bump-v0", "0.02"])
        flat = man.flat()
        assert flat["bump_v0"] == 0.02 and flat["kappa"] == 6.21 and flat["format"] == "table"
        json.dumps(flat)

    def test_surface_grids(self):
        assert cli.parse_grid("80:121:5") == [80.0, 85.0, 90.0, 95.0, 100.0, 105.0, 110.0, 115.0, 120.0]
        assert cli.parse_grid("0.25,0.5") == [0.25, 0.5]
        _, _, merged = parse_config(["surface", "--strikes", "90,100", "--maturities", "0.5,1"])
        assert merged["_strikes"] == [90.0, 100.0] and merged["_maturities"] == [0.5, 1.0]



class TestUsageErrors:
    """All rejected on the host before any device work: exit code 2."""

    @pytest.mark.parametrize("argv,needle", [
        (["price", "--rho", "1.5"], "rho"),
        (["price", "--paths", "0"], "n_paths"),
        (["price", "--scheme", "milstein", "--sampler", "sobol"], "sobol"),
        (["greeks", "--right", "put"], "call"),
        (["bench", "--scheme", "heun"], "heun"),
        (["price", "--scheme", "milstein", "--product", "asian", "--averaging-times", "0.3",
          "--steps", "16"], "grid"),
    ])
    def test_exit_code_2(self, capsys, argv, needle):
        code, _, err = run(capsys, argv)
        assert code == 2 and needle in err.lower()

    def test_unknown_config_key(self, tmp_path, capsys):
        f = tmp_path / "cfg.txt"
        f.write_text("bogus = 1\n")
        code, _, err = run(capsys, ["price", "--config", str(f)])
        assert code == 2 and "bogus" in err

    def test_bad_config_value(self, tmp_path, capsys):
        f = tmp_path / "cfg.txt"
        f.write_text("paths = many\n")
        code, _, err = run(capsys, ["price", "--config", str(f)])
        assert code == 2


@pytest.mark.gpu
class TestOutputs:
    def test_table(self, capsys):
        code, out, _ = run(capsys, ["price"] + FAST)
        assert code == 0 and out.startswith("# manifest ") and "price" in out

    def test_csv_round_trip(self, capsys):
        code, out, err = run(capsys, ["greeks", "--format", "csv"] + FAST)
        assert code == 0 and err.startswith("# manifest ")
        lines = out.strip().splitlines()
        assert lines[0] == "quantity," + CSV_HEADER
        names = [ln.split(",")[0] for ln in lines[1:]]
        assert names == ["price", "delta", "rho"]          # the reference's rows
        code, out, err = run(capsys, ["greeks", "--format", "csv", "--full-greeks"] + FAST)
        names = [ln.split(",")[0] for ln in out.strip().splitlines()[1:]]
        assert code == 0 and names == ["price", "delta", "gamma", "vega", "rho", "delta_fd", "rho_fd"]

    def test_exact_default_scheme(self, capsys):
        # the reference's default invocation: exact scheme, sobol, 256 paths
        code, out, _ = run(capsys, ["price", "--paths", "256", "--runs", "2", "--sampler", "sobol"])
        assert code == 0 and "price" in out

    def test_jsonl(self, capsys):
        code, out, _ = run(capsys, ["price", "--format", "jsonl", "--precision", "fp64"] + FAST)
        row = json.loads(out.strip().splitlines()[0])
        assert code == 0 and row["quantity"] == "price" and row["precision"] == "fp64"
        assert row["mean"] > 0

    def test_bridge_flags(self, capsys):
        code, out, _ = run(capsys, ["greeks", "--format", "jsonl", "--scheme", "milstein", "--sampler",
                                    "sobol", "--sobol-highdim-ack", "--sobol-scramble", "--sobol-bridge",
                                    "16", "--paths", "4096", "--steps", "64", "--runs", "4"])
        row = json.loads(out.strip().splitlines()[0])
        assert code == 0 and row["sobol_bridge"] == 16 and row["quantity"] == "price"
        assert abs(row["mean"] - 6.8) < 0.2

    def test_surface_csv(self, capsys):
        code, out, _ = run(capsys, ["surface", "--strikes", "90:111:10", "--maturities", "0.5,1",
                                    "--steps", "32", "--paths", "8192", "--runs", "2", "--s0", "100",
                                    "--scheme", "milstein"])
        lines = out.strip().splitlines()
        assert code == 0 and lines[0].startswith("style,maturity,strike,quantity")
        assert len(lines) == 1 + 2 * 7 * 2 * 3

    def test_bench_sweep_and_points(self, capsys, tmp_path):
        pts = tmp_path / "pts.csv"
        code, out, _ = run(capsys, ["bench", "--scheme", "euler,milstein", "--paths", "2048",
                                    "--steps", "8,16", "--runs", "3", "--emit-points", str(pts)])
        lines = out.strip().splitlines()
        assert code == 0 and lines[0] == CSV_HEADER and len(lines) == 5
        body = pts.read_text().splitlines()
        assert body[0] == "sampler,x,y" and len(body) == 1 + 2 * 1024
        import oracle   # the pseudo pairs are the reference stream keyed root_key(seed)
        want = oracle.uniforms_at(oracle.root_key(0), 0, 4)
        got = [float(v) for ln in body[1:3] for v in ln.split(",")[1:]]
        assert got == [float(f"{x:.10g}") for x in want]
