"""Orchestration/output row: traffic model, CSV/VTK formats
and the CLI (CPU parts; the GPU run is marked)."""

import csv
from fractions import Fraction

import numpy as np
import pytest

from paper_2408_06880_b200 import cli, geometry, model, output
from paper_2408_06880_b200.model import TrafficModel


def test_byte_counts_and_reductions_match_the_reference_model():
    # reference tests/test_acceptance.py:89-125 (criterion 01)
    want = {("cpu", "dense", "pull"): 456, ("cpu", "sparse", "pull"): 528,
            ("cpu", "dense", "aa"): 304, ("cpu", "sparse", "aa"): 340,
            ("gpu", "dense", "pull"): 304, ("gpu", "sparse", "pull"): 376,
            ("gpu", "dense", "aa"): 304, ("gpu", "sparse", "aa"): 340}
    for (arch, s, p), b in want.items():
        assert model.bytes_per_cell(TrafficModel(arch, s, p, 19, 8, 4)) == b
    assert model.traffic_reduction("gpu", "sparse", 19) == Fraction(9, 94)
    assert model.traffic_reduction("cpu", "sparse", 19) == Fraction(47, 132)
    assert model.aa_memory_saving(19) == Fraction(152, 416)
    assert model.memory_breakeven(19) == Fraction(344, 416)


def test_csv_schema(tmp_path):
    p = tmp_path / "r.csv"
    output.write_csv_records([{"run_id": "a", "steps": 3, "elapsed_s": 0.5}], p)
    rows = list(csv.reader(open(p)))
    assert rows[0] == output.CSV_COLUMNS + output.WALLCLOCK_COLUMNS
    assert rows[1][0] == "a" and rows[1][-2] == "0.5"
    with pytest.raises(ValueError):
        output.write_csv_records([{"bogus": 1}], p)


def test_cli_exit_codes_and_info(tmp_path, capsys):
    assert cli.main(["info", "--q", "27"]) == 0
    assert "Q=27" in capsys.readouterr().out
    assert cli.main(["run", "--bogus"]) == cli.EXIT_USAGE
    assert cli.main(["run", "--policy", "weird"]) == cli.EXIT_CONFIG
    assert cli.main(["run", "--overlap", "maybe"]) == cli.EXIT_CONFIG
    cfgf = tmp_path / "c.cfg"
    cfgf.write_text("steps = 3\nnot a pair\n")
    assert cli.main(["run", "--config", str(cfgf)]) == cli.EXIT_CONFIG
    assert cli.main(["convert", "preview", "--mask", str(tmp_path / "missing.svx")]) == cli.EXIT_IO


def test_cli_convert_bed_and_preview(tmp_path):
    m = tmp_path / "bed.svx"
    assert cli.main(["convert", "bed", "--extent", "20,16,12", "--porosity", "0.6",
                     "--out-path", str(m)]) == 0
    mask = geometry.read_voxel_mask(m)
    assert mask.dims == (20, 16, 12) and 0.45 < mask.porosity() < 0.75
    v = tmp_path / "bed.vtk"
    assert cli.main(["convert", "preview", "--mask", str(m), "--out-path", str(v)]) == 0
    solid = output.read_vtk_scalars(v, "solid")
    assert np.array_equal(solid.astype(bool), mask.solid)


@pytest.mark.gpu
def test_cli_run_and_sweep_on_gpu(tmp_path, gpu_lib):
    rc = cli.main(["run", "--geometry", "riverbed", "--dims", "16,16", "--block-size", "8,8",
                   "--pattern", "aa", "--overlap", "on", "--steps", "6", "--vtk", "on",
                   "--policy", "hybrid", "--out", str(tmp_path), "--run-id", "t"])
    assert rc == 0
    row = list(csv.DictReader(open(tmp_path / "t.csv")))[0]
    assert row["steps"] == "6" and int(row["messages"]) > 0
    rho = output.read_vtk_scalars(tmp_path / "t.block0000.vtk", "density")
    assert rho.shape == (1, 8, 8) and rho.max() > 0.9  # 2-D block: DIMENSIONS 8 8 1
    rc = cli.main(["sweep-porosity", "--dims", "24,24,24", "--stencil", "D3Q19", "--steps", "4",
                   "--phis", "0.5,1.0", "--pattern", "aa", "--out", str(tmp_path)])
    assert rc == 0
    rows = list(csv.DictReader(open(tmp_path / "sweep.csv")))
    assert len(rows) == 6 and {r["layout"] for r in rows} == {"sparse", "dense", "hybrid"}
