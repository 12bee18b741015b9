#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03_final3_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_final3_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03_final3_smoke.txt 2>&1
timeout 400 python bench.py > gpurun_out/r03_final3_bench.json 2> gpurun_out/r03_final3_bench.err
