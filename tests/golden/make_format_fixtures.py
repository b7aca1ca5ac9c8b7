"""Hand-derived interop fixtures for the two file formats either side of the hot path.

The reference cannot emit these files in this environment: `src/landmarks.cpp` needs Eigen and
`src/registration.cpp` needs nlohmann/json.hpp plus template deductions that do not compile.
So the fixtures are derived from the reference SOURCE, field by field, by this script -- which deliberately does
not import the package under test:

  reference_landmarks_3d.txt   what save_landmarks (landmarks.cpp:123-140) writes: one landmark per line,
                               every coordinate printed with "%.17g" (snprintf), single blanks, '\n' line ends.
                               The strings are written out literally below and cross-checked against libc's
                               printf through Python's % operator.
  reference_result_v1.json     what save_result (registration.cpp:207-260) writes: `doc.dump(2)` of a
                               nlohmann::json object = keys in sorted order (std::map), two-space indent, every
                               array element on its own line, `"key": value`, floats in shortest round-trip form with
                               a trailing ".0" for integral values, a final '\n'.  Enum strings: the reference
                               declares to_string(Precision / ReduceStrategy / StopReason) but ships no definition
                               (shooting.hpp:19-20, reduction.hpp:213-214); the enumerator names are used
                               (f32|f64, sequential|precompute_matrix|blocked_tree,
                               gradient_tolerance|max_iterations|line_search_failure).

The result document describes a registration whose numbers follow in closed form (the N = 1 flight is
exact): two landmarks 1000 mm apart with sigma = 1.5 (K_12 = exp(-1e6/4.5) underflows to exactly 0, K_ii = 1), so
each moves in a straight line: warped = template + momenta (T = 4, dt = 1/4: exact in binary).
  H = 1/2 (|p_1|^2 + |p_2|^2) = 1/2 (1.3125 + 1.3125) = 1.3125;  mismatch = |warped - target|^2 = 0.25;
  final_loss = H + lambda * mismatch = 1.3125 + 10 * 0.25 = 3.8125
  initial p0 = (target - template)/T  ->  q(1) = template + (target - template)/4, mismatch = (3/4)^2 (2.5625 + 1.3125)
  = 2.1796875, H = 1/2 (2.5625 + 1.3125)/16 = 0.12109375, initial_loss = 0.12109375 + 21.796875 = 21.91796875
  distances before: sqrt(2.5625), sqrt(1.3125); after: 0.5, 0.
The per-iteration history entries are illustrative (load_result, registration.cpp:262-308, does not read them).
"""
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))

# ---- landmark text ---------------------------------------------------------------------------------------
LANDMARK_ROWS = [
    ("0.10000000000000001 1.5 -2", (0.1, 1.5, -2.0)),
    ("1.0000000000000001e-09 123456789.125 0.33333333333333331", (1e-9, 123456789.125, 1.0 / 3.0)),
    ("25000000000 -0 6.0221407599999999e+23", (2.5e10, -0.0, 6.02214076e23)),
    ("-17.25 3.1415926535897931 2.2250738585072014e-308", (-17.25, math.pi, 2.2250738585072014e-308)),
]
for line, vals in LANDMARK_ROWS:
    assert line == " ".join("%.17g" % v for v in vals), (line, vals)
with open(os.path.join(HERE, "reference_landmarks_3d.txt"), "w", newline="") as f:
    f.write("".join(line + "\n" for line, _ in LANDMARK_ROWS))

# ---- result document ---------------------------------------------------------------------------------------
d1, d2 = math.sqrt(2.5625), math.sqrt(1.3125)
DOC = {
    "config": {"backend": "blocked_tree", "block_size": 256, "lambda": 10.0, "max_iter": 2, "precision": "f64",
               "procrustes": False, "seed": 0, "sigma": 1.5, "threads": 0, "timesteps": 4},
    "history": {"evaluations": 3, "final_loss": 3.8125, "grad_inf_norm": [4.0, 1.0], "initial_loss": 21.91796875,
                "iterations": 2, "loss": [7.5, 3.8125], "step": [1.0, 1.0], "stop_reason": "max_iterations"},
    "metrics": {"avg_after_mm": 0.25, "avg_before_mm": (d1 + d2) / 2.0, "max_after_mm": 0.5, "max_before_mm": d1},
    "momenta": [0.5, -0.25, 1.0, -1.0, 0.5, 0.25],
    "points": {"count": 2, "dim": 3,
               "target": [[1.5, 1.75, 4.5], [1000.0, 2.5, 3.25]],
               "template": [[1.0, 2.0, 3.0], [1001.0, 2.0, 3.0]],
               "warped": [[1.5, 1.75, 4.0], [1000.0, 2.5, 3.25]]},
    "schema_version": 1,
    "timing": {"note": "wall times are environment-dependent", "per_gradient_mean_seconds": 0.125, "total_seconds": 0.5},
}


def emit(v, indent):
    """nlohmann::json::dump(2) for the value kinds save_result produces."""
    pad, inner = " " * indent, " " * (indent + 2)
    if isinstance(v, dict):
        items = [f'{inner}"{k}": {emit(v[k], indent + 2)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(inner + emit(e, indent + 2) for e in v) + "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        r = repr(v)  # shortest round-trip digits, as nlohmann's Grisu2 (identical for the magnitudes used here)
        return r if any(c in r for c in ".en") else r + ".0"
    if isinstance(v, str):
        return '"' + v + '"'
    raise TypeError(v)


with open(os.path.join(HERE, "reference_result_v1.json"), "w", newline="") as f:
    f.write(emit(DOC, 0) + "\n")
