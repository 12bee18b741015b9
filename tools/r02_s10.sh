args=""
for t in TILE_C_8 TILE_C_2 DESCEND_UNROLL_2 CARVEOUT_0 CARVEOUT_25 APPROX_NORM_1 DYN_MINBLOCKS_9; do args="$args 'run $t FGL_LIB=build_ab/libfgl_FGL_$t.so'"; done
eval MODE=cast bash tools/sweep.sh "'run base'" $args "'run base2'" > gpurun_out/r02_s10_sweep.txt 2>&1
eval BENCH_ARGS=\"--config C5 --poses 256\" MODE=cast bash tools/sweep.sh "'run c5base'" "'run c5TILE_C_2 FGL_LIB=build_ab/libfgl_FGL_TILE_C_2.so'" "'run c5APPROX_NORM_1 FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so'" >> gpurun_out/r02_s10_sweep.txt 2>&1
