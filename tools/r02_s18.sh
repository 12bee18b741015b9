python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.txt 2>&1
for cfg in G2 T2; do python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/r02_configs_next.jsonl; done
