"""Host-side pieces of the stability-sweep harness (experiments.py mirror):
validation, sampled widths, the input generator and the byte format of the
CSV writer, pinned by the reference's own output (tests/golden, written by
tests/golden/make_golden.py from the unmodified reference)."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_2405_10923_b200 import experiments as E


def test_sample_widths():
    # experiments.py:101-105 (test_experiments.py:34-38)
    assert E.sample_widths(300, 25) == list(range(25, 301, 25))
    assert E.sample_widths(10, 3) == [3, 6, 9, 10]
    assert E.sample_widths(5, 10) == [5]
    assert E.sample_widths(8, 8) == [8]


def test_config_validation():
    with pytest.raises(ValueError):
        E.ExperimentConfig(algo="mgs", every=0)
    with pytest.raises(ValueError):
        E.ExperimentConfig(algo="mgs", ell=-4)
    with pytest.raises(ValueError):
        E.run_factor_experiment(np.eye(4), E.ExperimentConfig(algo="qr-but-wrong"))
    with pytest.raises(NotImplementedError):
        E.run_factor_experiment(np.eye(4), E.ExperimentConfig(algo="mgs"))
    with pytest.raises(ValueError):
        E.run_gmres_experiment(np.eye(4), np.ones(4), 2, E.ExperimentConfig(algo="hqr"))
    with pytest.raises(NotImplementedError):
        E.run_gmres_experiment(np.eye(4), np.ones(4), 2, E.ExperimentConfig(algo="rgs"))


def test_gen_cmatrix_bitwise_and_corners():
    g = golden("experiments_cmatrix_2048x48")
    W = E.gen_cmatrix(2048, 48)
    assert hashlib.sha256(np.ascontiguousarray(W).tobytes()).hexdigest() == str(g["W_sha"])
    C = E.gen_cmatrix(5, 5)  # test_experiments.py:16-23
    assert C[0, 0] == 0.0 and C[-1, -1] == np.sin(20.0) / 2.1
    with pytest.raises(ValueError):
        E.gen_cmatrix(1, 5)


def _rows(g, name, cls):
    return [cls(int(j), *map(float, v), str(s))
            for j, v, s in zip(g[f"{name}_j"], g[f"{name}_vals"], g[f"{name}_status"])]


@pytest.mark.parametrize("name", ["left", "right", "block", "rec", "leftgauss", "mixed"])
def test_csv_bytes_match_reference(tmp_path, name):
    g = golden("experiments_cmatrix_2048x48")
    rows = _rows(g, name, E.MetricRow)
    cfg_line = bytes(g[f"{name}_csv"]).decode().splitlines()[0]
    # rebuild the config the reference echoed, then write the same rows
    cfg = eval(cfg_line[2:], {"ExperimentConfig": E.ExperimentConfig})  # noqa: S307 (our own fixture)
    p = tmp_path / "out.csv"
    E.write_csv(str(p), rows, config=cfg, extra="golden")
    assert p.read_bytes() == bytes(g[f"{name}_csv"])


def test_gmres_csv_bytes_match_reference(tmp_path):
    g = golden("experiments_gmres_cd24")
    rows = _rows(g, "srht", E.GmresRow)
    cfg = E.ExperimentConfig(algo="rhqr", seed=4, deterministic=True)
    p = tmp_path / "g.csv"
    E.write_csv(str(p), rows, config=cfg, extra="golden")
    assert p.read_bytes() == bytes(g["srht_csv"])


def test_csv_timestamp_unless_deterministic(tmp_path):
    rows = [E.MetricRow(4, 1.0, 1.0, 0.0, 0.0, 0.0, "ok")]
    c = tmp_path / "c.csv"
    E.write_csv(str(c), rows, config=E.ExperimentConfig(algo="rhqr-left"))
    assert any(ln.startswith("# written") for ln in c.read_text().splitlines())
