# refresh config 2's judged artefacts after the swizzled R == 1 bitmap (into gpurun_out/m2, then tools/ingest_m2.sh)
O=gpurun_out/m2; mkdir -p $O; T="timeout 900"; c=2
$T python bench.py --config $c > $O/bench_cfg$c.log 2>&1
$T python bench.py --config $c --cap 300 --no-accuracy > $O/bench_cfg${c}_cap300.log 2>&1
$T python bench.py --impl reference --config $c > $O/ref_cfg$c.log 2>&1
$T ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv python bench.py --config $c --profile-steps 1 > /dev/null 2>&1
$T ncu --set full --clock-control none --import-source on -k "regex:k_degree|k_tile_rows|k_flop" -o $O/flop_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/flop_cfg$c.log 2>&1
$T ncu --set full --clock-control none --import-source on -k "regex:k_predict|k_sym_block_hash|k_heavy_run|k_heavy_sort" -o $O/symp_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/symp_cfg$c.log 2>&1
