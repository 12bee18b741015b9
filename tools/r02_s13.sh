python tools/pcie_bw.py > gpurun_out/r02_pcie.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_par3.csv python bench.py --restructure -3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_par3.csv > gpurun_out/r02_launches_par3.txt 2>&1
