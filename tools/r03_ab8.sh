#!/bin/bash
mkdir -p gpurun_out
MODE=full bash tools/sweep.sh 'run plain' 'run b11 -- --morton-bits 11' 'run b12 -- --morton-bits 12' 'run b13 -- --morton-bits 13' 'run box1 -- --morton-box 1' 'run b9 -- --morton-bits 9' > gpurun_out/r03_ab8.txt 2>&1
