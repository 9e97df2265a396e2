"""f2 — binary score files (rw_write_scores_f64 / rw_read_scores_f64): the
reference ingests scores as CSV (load_scores, workload.cpp:32-62); the .f64 path is one read,
bit-exact, and validated like ScoreMatrix::validate (workload.cpp:23-29).  CPU only."""
import os

import numpy as np
import pytest

import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import routeplan as rp


def test_round_trip_bit_exact(tmp_path):
    s = rw.synth_scores(5000, ["A", "B", "C", "D"], [(2, 8), (4, 6), (6, 4), (8, 2)], 7)
    p = str(tmp_path / "s.f64")
    rp.write_scores_f64(s, p)
    t = rp.read_scores_f64(p)
    assert t.models == ["A", "B", "C", "D"]
    assert t.scores.shape == (5000, 4)
    assert np.array_equal(t.scores.view(np.int64), s.scores.view(np.int64))
    # header (8) + n, m (16) + names (4 x (4 + 1)) + data
    assert os.path.getsize(p) == 8 + 16 + 4 * 5 + 5000 * 4 * 8


def test_out_of_range_entry_is_validation_error(tmp_path):
    s = rw.synth_scores(10, ["A", "B"], [(2, 8), (8, 2)], 1)
    s.scores[3, 1] = 1.5
    p = str(tmp_path / "bad.f64")
    rp.write_scores_f64(s, p)
    with pytest.raises(rp.ValidationError, match=r"prompt 'p4', model 'B' is 1.5, outside \[0, 1\]"):
        rp.read_scores_f64(p)


def test_missing_or_foreign_file_is_config_error(tmp_path):
    with pytest.raises(rp.ConfigError):
        rp.read_scores_f64(str(tmp_path / "nope.f64"))
    p = tmp_path / "csv.f64"
    p.write_text("prompt_id,A\np1,0.5\n")
    with pytest.raises(rp.ConfigError, match="not a RWSCORE1"):
        rp.read_scores_f64(str(p))
