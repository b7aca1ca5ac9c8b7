"""The data formats either side of the hot path: landmark text files
(landmarks.cpp:59-140) and the schema-v1 JSON result document (registration.cpp:203-308).  CPU only."""
import json

import numpy as np
import pytest

from paper_1907_04839_b200 import (IoError, ParseError, ResultDocument, ShapeError, ShootingConfig, load_landmarks,
                                   load_result, save_landmarks, save_result)


def test_landmark_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(3)
    for dim in (2, 3):
        pts = rng.normal(size=(57, dim)) * np.array([1e-9, 1.0, 1e9][:dim])
        path = tmp_path / f"pts{dim}.txt"
        save_landmarks(pts, path)
        back = load_landmarks(path)
        assert back.shape == pts.shape and np.array_equal(back, pts)  # %.17g round-trips every double
        assert all(len(line.split(" ")) == dim for line in path.read_text().splitlines())


def test_landmark_parser_accepts_reference_separators_and_comments(tmp_path):
    path = tmp_path / "mixed.txt"
    path.write_text("# header\n\n  1.5, 2.5,\t-3e1  # trailing comment\r\n4 5 6\r\n   \n#only comment\n.5,-.25,1.\n")
    pts = load_landmarks(path)
    assert np.array_equal(pts, [[1.5, 2.5, -30.0], [4, 5, 6], [0.5, -0.25, 1.0]])
    assert load_landmarks(path, expected_dim=3).shape == (3, 3)
    with pytest.raises(ShapeError):
        load_landmarks(path, expected_dim=2)


@pytest.mark.parametrize("text, line, what", [
    ("1 2 3\n4 5\n", 2, "inconsistent field count"),
    ("1 2 3 4\n", 1, "expected 2 or 3 fields"),
    ("1\n", 1, "expected 2 or 3 fields"),
    ("1 2 3\n4 abc 6\n", 2, "non-numeric token 'abc 6'"),
    ("1 2 +3\n", 1, "non-numeric token"),          # std::from_chars takes no leading plus
    ("1 2 3\n\n1 nan 3\n", 3, "non-finite coordinate"),
    ("1 -inf\n", 1, "non-finite coordinate"),
    ("1 2e\n", 1, "non-numeric token 'e'"),
])
def test_landmark_parse_errors_carry_the_line(tmp_path, text, line, what):
    path = tmp_path / "bad.txt"
    path.write_text(text)
    with pytest.raises(ParseError) as e:
        load_landmarks(path)
    assert e.value.line == line and what in str(e.value) and f"at line {line}" in str(e.value)


def test_landmark_file_errors(tmp_path):
    with pytest.raises(IoError):
        load_landmarks(tmp_path / "missing.txt")
    empty = tmp_path / "empty.txt"
    empty.write_text("# nothing here\n\n")
    with pytest.raises(ParseError) as e:
        load_landmarks(empty)
    assert e.value.line == 0 and "no landmarks" in str(e.value)
    with pytest.raises(IoError):
        save_landmarks(np.zeros((2, 3)), tmp_path / "no_such_dir" / "x.txt")


def _doc():
    rng = np.random.default_rng(5)
    n = 9
    return ResultDocument(
        config=ShootingConfig(sigma=1.25, timesteps=7, lam=123.5, max_iter=33, precision="f32"),
        procrustes_applied=True, template=rng.normal(size=(n, 3)), target=rng.normal(size=(n, 3)),
        warped=rng.normal(size=(n, 3)), momenta=rng.normal(size=n * 3) * 1e-7, avg_before=1.7439, max_before=5.7804,
        avg_after=0.089, max_after=0.469, initial_loss=8.16e8, final_loss=1478.16, stop_reason="gradient_tolerance",
        evaluations=105, hist_loss=[3.0, 2.0, 1.0], hist_grad_inf_norm=[0.3, 0.2, 0.1], hist_step=[1.0, 0.5, 1.0],
        total_seconds=27.0, eval_seconds_mean=0.25)


def test_result_document_layout_is_the_reference_schema(tmp_path):
    path = tmp_path / "result.json"
    save_result(_doc(), path)
    raw = json.loads(path.read_text())
    # sections and keys exactly as save_result writes them (registration.cpp:207-252)
    assert list(raw) == sorted(raw) and set(raw) == set(["schema_version", "config", "metrics", "history", "momenta", "points", "timing"])  # nlohmann sorts keys
    assert raw["schema_version"] == 1
    assert set(raw["config"]) == set(["sigma", "timesteps", "lambda", "max_iter", "precision", "backend", "block_size",
                                   "threads", "seed", "procrustes"])
    assert set(raw["metrics"]) == set(["avg_before_mm", "max_before_mm", "avg_after_mm", "max_after_mm"])
    assert set(raw["history"]) == set(["initial_loss", "stop_reason", "iterations", "evaluations", "loss",
                                    "grad_inf_norm", "step", "final_loss"])
    assert raw["history"]["iterations"] == 3
    assert set(raw["points"]) == set(["dim", "count", "template", "target", "warped"])
    assert raw["points"]["dim"] == 3 and raw["points"]["count"] == 9 and len(raw["points"]["warped"][0]) == 3
    assert set(raw["timing"]) == set(["note", "total_seconds", "per_gradient_mean_seconds"])
    assert len(raw["momenta"]) == 27


def test_result_document_round_trip_is_exact(tmp_path):
    doc = _doc()
    path = tmp_path / "result.json"
    save_result(doc, path)
    back = load_result(path)
    # "Momenta and points round-trip exactly" (registration.hpp:61-62)
    for name in ("template", "target", "warped", "momenta"):
        assert np.array_equal(getattr(back, name), getattr(doc, name)), name
    assert back.config == doc.config and back.procrustes_applied
    assert (back.avg_before, back.max_before, back.avg_after, back.max_after) == (1.7439, 5.7804, 0.089, 0.469)
    assert back.final_loss == doc.final_loss and back.evaluations == 105 and back.hist_loss == [3.0, 2.0, 1.0]


def test_result_document_errors(tmp_path):
    with pytest.raises(IoError):
        load_result(tmp_path / "missing.json")
    bad = tmp_path / "bad.json"
    bad.write_text("{ not json")
    with pytest.raises(ParseError):
        load_result(bad)
    path = tmp_path / "result.json"
    save_result(_doc(), path)
    raw = json.loads(path.read_text())
    other = dict(raw, schema_version=2)
    bad.write_text(json.dumps(other))
    with pytest.raises(ParseError, match="unsupported result schema version"):
        load_result(bad)
    for section, key in (("config", "sigma"), ("metrics", "max_after_mm"), ("history", "final_loss"), ("points", "dim")):
        broken = json.loads(path.read_text())
        del broken[section][key]
        bad.write_text(json.dumps(broken))
        with pytest.raises(ParseError, match="missing fields"):
            load_result(bad)
    broken = json.loads(path.read_text())
    del broken["momenta"]
    bad.write_text(json.dumps(broken))
    with pytest.raises(ParseError, match="missing fields"):
        load_result(bad)
