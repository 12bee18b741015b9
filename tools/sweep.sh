#!/bin/bash
# A/B sweep of cast-kernel variants on the C2 workload (run under gpurun); one line per variant.
# run label [ENV=val ...] [-- extra bench args]
run() {
  local label=$1; shift
  local envs=() extra=()
  while [ $# -gt 0 ]; do
    if [ "$1" = "--" ]; then shift; extra=("$@"); break; fi
    envs+=("$1"); shift
  done
  out=$(env "${envs[@]}" python bench.py --mode ${MODE:-full} --steps 20 --warmup 3 --no-cpu --no-e2e --no-latency $BENCH_ARGS "${extra[@]}" 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print(f\"{sys.argv[2]:28s} cast {d['cast_rays_per_s']/1e9:6.3f} Grays/s  {d['cast_ms']:.3f} ms  nodes {d['nodes_per_ray']:.1f} tris {d['tris_per_ray']:.1f} build {d['build_ms']:.3f} ms full {d['value']/1e9:.3f}\")" "$out" "$label"
}
for v in "$@"; do eval "$v"; done
