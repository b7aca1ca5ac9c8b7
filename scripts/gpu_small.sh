#!/bin/bash
# Persistent small-N kernel: parity tests that exercise it, then the persistent-vs-tiled A/B.  usage: gpu_small.sh [tag]
tag=${1:-small}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "persistent or compute_gradient_parity or determinism or golden or hundred or extension" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${tag}_pytest.log
timeout 600 python scripts/small_ab.py gpurun_out/${tag}_small_ab.json 500 1000 1500 2000 2500 3000 3500 4000 > gpurun_out/${tag}_small_ab.log 2>&1; python - <<PY
import json
for r in json.load(open("gpurun_out/${tag}_small_ab.json")):
    print(r["n"], r["precision"], "persistent %.4f ms (%d launches, frac %.3f) | tiled %.4f ms" % (r["persistent"]["device_ms"], r["persistent"]["launches"], r["persistent"]["roofline_frac"], r["tiled"]["device_ms"]))
PY
timeout 300 python scripts/gpu_c1.py > gpurun_out/${tag}_c1.log 2>&1; cat gpurun_out/${tag}_c1.log
if [ -f paper_1907_04839_b200/liblmshoot_b200_trace.so ]; then LMS_LIB_PATH=paper_1907_04839_b200/liblmshoot_b200_trace.so timeout 300 python scripts/small_trace.py 1000 2000 4000 2>&1 | grep -v "f64: device.*e+\|[0-9]\{12\}" ; fi
