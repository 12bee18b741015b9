#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r03_final4_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_final4_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03_final4_smoke.txt 2>&1
