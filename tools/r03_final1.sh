#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03_final1_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_final1_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_final1_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_final1_build_ms.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03_final1_smoke.txt 2>&1
