#!/bin/bash
mkdir -p gpurun_out
MODE=full bash tools/sweep.sh 'run b10 -- --morton-bits 10' 'run b8 -- --morton-bits 8' 'run b7 -- --morton-bits 7' > gpurun_out/r03_ab9.txt 2>&1
BENCH_ARGS="--config C5 --poses 128" MODE=full bash tools/sweep.sh 'run c5b13' 'run c5b10 -- --morton-bits 10' 'run c5b8 -- --morton-bits 8' >> gpurun_out/r03_ab9.txt 2>&1
BENCH_ARGS="--config C4" MODE=full bash tools/sweep.sh 'run c4b10' 'run c4b8 -- --morton-bits 8' >> gpurun_out/r03_ab9.txt 2>&1
