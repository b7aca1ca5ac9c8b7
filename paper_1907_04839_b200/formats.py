"""The data formats either side of the hot path: the landmark text format
(landmarks.cpp:59-140) and the versioned JSON result document (registration.cpp:203-308), so that files
written by the reference's tooling load here and the other way round.

Nothing here touches the GPU; the arithmetic-free parsing rules follow the reference line by line:
separators are blanks, tabs, commas and carriage returns; `#` starts a comment; the first data line fixes
the dimension (2 or 3); every coordinate must be finite; coordinates are written with 17 significant
digits so a load/save cycle is exact.
"""
from __future__ import annotations

import json
import math
import os
import re
from dataclasses import dataclass, field

import numpy as np

from .errors import IoError, ParseError, ShapeError
from .shooting import ShootingConfig

SCHEMA_VERSION = 1  # registration.cpp:203

# std::from_chars(double) grammar (landmarks.cpp:72): optional minus (no plus), digits with an optional
# fraction or a bare fraction, optional exponent; or inf / nan (rejected afterwards as non-finite).
_NUMBER = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)", re.IGNORECASE)
_SEPARATORS = " \t,\r"


def _parse_line_fields(line: str, line_no: int) -> list[float]:
    """parse_line_fields (landmarks.cpp:61-81)."""
    fields = []
    p, end = 0, len(line)
    while p < end:
        while p < end and line[p] in _SEPARATORS:
            p += 1
        if p >= end or line[p] == "#":  # trailing comment
            break
        m = _NUMBER.match(line, p)
        if not m:
            raise ParseError(f"non-numeric token '{line[p:p + 16]}'", line_no)
        tok = m.group(0)
        fields.append(float("nan") if "nan" in tok.lower() else float(tok))
        p = m.end()
    return fields


def load_landmarks(path, expected_dim: int | None = None) -> np.ndarray:
    """load_landmarks (landmarks.cpp:85-121) -> (n, dim) float64."""
    try:
        fh = open(path, "r", newline="")
    except OSError as e:
        raise IoError(f"cannot open landmark file: {path}") from e
    coords: list[float] = []
    dim = 0
    with fh:
        for line_no, raw in enumerate(fh.read().split("\n"), start=1):
            stripped = raw.lstrip(" \t\r")
            if not stripped or stripped[0] == "#":
                continue
            fields = _parse_line_fields(raw, line_no)
            if not fields:
                continue
            if dim == 0:
                if len(fields) not in (2, 3):
                    raise ParseError(f"expected 2 or 3 fields, found {len(fields)}", line_no)
                dim = len(fields)
            elif len(fields) != dim:
                raise ParseError(f"inconsistent field count (expected {dim}, found {len(fields)})", line_no)
            for v in fields:
                if not math.isfinite(v):
                    raise ParseError("non-finite coordinate", line_no)
                coords.append(v)
    if not coords:
        raise ParseError(f"no landmarks in {path}")
    if expected_dim is not None and dim != expected_dim:
        raise ShapeError(f"expected dimension {expected_dim}, file {path} has dimension {dim}")
    return np.asarray(coords, dtype=np.float64).reshape(-1, dim)


def save_landmarks(points, path) -> None:
    """save_landmarks (landmarks.cpp:123-140): one landmark per line, `%.17g`, single blanks."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise ShapeError("save_landmarks: expected an (n, dim) array")
    try:
        with open(path, "w", newline="") as fh:
            for row in pts:
                fh.write(" ".join("%.17g" % v for v in row) + "\n")
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


@dataclass
class ResultDocument:
    """RegistrationResult as stored (registration.hpp:28-46).  The CPU-only configuration fields the
    reference writes (backend, block_size, threads, seed) are carried through unchanged so that a
    reference-written document survives a load/save cycle here."""

    config: ShootingConfig = field(default_factory=ShootingConfig)
    procrustes_applied: bool = False
    backend: str = "blocked_tree"   # ReduceStrategy (reduction.hpp:27-31); this build's kernels have no such switch
    block_size: int = 256
    threads: int = 0
    seed: int = 0
    template: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    target: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    warped: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    momenta: np.ndarray = field(default_factory=lambda: np.zeros(0))  # flat N*dim, registration.hpp:36
    avg_before: float = 0.0
    max_before: float = 0.0
    avg_after: float = 0.0
    max_after: float = 0.0
    initial_loss: float = 0.0
    final_loss: float = 0.0
    stop_reason: str = "max_iterations"
    evaluations: int = 0
    hist_loss: list = field(default_factory=list)
    hist_grad_inf_norm: list = field(default_factory=list)
    hist_step: list = field(default_factory=list)
    total_seconds: float = 0.0
    eval_seconds_mean: float = 0.0


def result_document_from(reg, template, target, config: ShootingConfig, total_seconds=0.0,
                         eval_seconds_mean=0.0) -> ResultDocument:
    """A ResultDocument from this package's register_landmarks() result (registration.cpp:81-98)."""
    return ResultDocument(
        config=config, template=np.asarray(template, dtype=np.float64), target=np.asarray(target, dtype=np.float64),
        warped=np.asarray(reg.warped, dtype=np.float64), momenta=np.asarray(reg.momenta, dtype=np.float64).ravel(),
        avg_before=reg.avg_before, max_before=reg.max_before, avg_after=reg.avg_after, max_after=reg.max_after,
        initial_loss=reg.initial_loss, final_loss=reg.final_loss, stop_reason=reg.reason,
        evaluations=reg.evaluations, hist_loss=[float(v) for v in reg.hist_loss],
        total_seconds=total_seconds, eval_seconds_mean=eval_seconds_mean)


def save_result(doc: ResultDocument, path) -> None:
    """save_result (registration.cpp:207-260): same sections, key names and nesting."""
    cfg = doc.config
    dim = int(doc.template.shape[1]) if doc.template.ndim == 2 and doc.template.size else 3
    out = {
        "schema_version": SCHEMA_VERSION,
        "config": {"sigma": cfg.sigma, "timesteps": cfg.timesteps, "lambda": cfg.lam, "max_iter": cfg.max_iter,
                   "precision": cfg.precision, "backend": doc.backend, "block_size": doc.block_size,
                   "threads": doc.threads, "seed": doc.seed, "procrustes": bool(doc.procrustes_applied)},
        "metrics": {"avg_before_mm": doc.avg_before, "max_before_mm": doc.max_before,
                    "avg_after_mm": doc.avg_after, "max_after_mm": doc.max_after},
        "history": {"initial_loss": doc.initial_loss, "stop_reason": doc.stop_reason,
                    "iterations": len(doc.hist_loss), "evaluations": doc.evaluations,
                    "loss": list(doc.hist_loss), "grad_inf_norm": list(doc.hist_grad_inf_norm),
                    "step": list(doc.hist_step), "final_loss": doc.final_loss},
        "momenta": [float(v) for v in np.asarray(doc.momenta).ravel()],
        "points": {"dim": dim, "count": int(len(doc.template)),
                   "template": np.asarray(doc.template).tolist(), "target": np.asarray(doc.target).tolist(),
                   "warped": np.asarray(doc.warped).tolist()},
        "timing": {"note": "wall times are environment-dependent", "total_seconds": doc.total_seconds,
                   "per_gradient_mean_seconds": doc.eval_seconds_mean},
    }
    try:
        with open(path, "w") as fh:
            # nlohmann::json keeps object keys sorted and dump(2) indents by two; floats round-trip exactly in both
            json.dump(out, fh, indent=2, sort_keys=True)
            fh.write("\n")
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def load_result(path) -> ResultDocument:
    """load_result (registration.cpp:262-308): IoError when unreadable, ParseError when corrupt, of another
    schema version, or missing any field the reference reads."""
    if not os.path.exists(path):
        raise IoError(f"cannot open result document: {path}")
    try:
        with open(path, "r") as fh:
            raw = json.load(fh)
    except OSError as e:
        raise IoError(f"cannot open result document: {path}") from e
    except json.JSONDecodeError as e:
        raise ParseError(f"corrupt result document {path}: {e}") from e
    try:
        if int(raw["schema_version"]) != SCHEMA_VERSION:
            raise ParseError(f"unsupported result schema version in {path}")
        c, m, h, pts = raw["config"], raw["metrics"], raw["history"], raw["points"]
        dim = int(pts["dim"])

        def points(rows):  # points_from_json, registration.cpp:194-201
            flat = [float(v) for row in rows for v in row]
            return np.asarray(flat, dtype=np.float64).reshape(-1, dim) if flat else np.zeros((0, dim))

        precision = str(c["precision"])
        if precision not in ("f32", "f64"):
            raise ParseError(f"unknown precision '{precision}' in {path}")
        return ResultDocument(
            config=ShootingConfig(sigma=float(c["sigma"]), timesteps=int(c["timesteps"]), lam=float(c["lambda"]),
                                  max_iter=int(c["max_iter"]), precision=precision),
            procrustes_applied=bool(c["procrustes"]), backend=str(c["backend"]), block_size=int(c["block_size"]),
            threads=int(c["threads"]), seed=int(c["seed"]),
            template=points(pts["template"]), target=points(pts["target"]), warped=points(pts["warped"]),
            momenta=np.asarray(raw["momenta"], dtype=np.float64),
            avg_before=float(m["avg_before_mm"]), max_before=float(m["max_before_mm"]),
            avg_after=float(m["avg_after_mm"]), max_after=float(m["max_after_mm"]),
            final_loss=float(h["final_loss"]),
            # the reference's loader stops here; the rest is kept when present
            initial_loss=float(h.get("initial_loss", 0.0)), stop_reason=str(h.get("stop_reason", "max_iterations")),
            evaluations=int(h.get("evaluations", 0)), hist_loss=list(h.get("loss", [])),
            hist_grad_inf_norm=list(h.get("grad_inf_norm", [])), hist_step=list(h.get("step", [])),
            total_seconds=float(raw.get("timing", {}).get("total_seconds", 0.0)),
            eval_seconds_mean=float(raw.get("timing", {}).get("per_gradient_mean_seconds", 0.0)))
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"result document {path} is missing fields: {e!r}") from e
