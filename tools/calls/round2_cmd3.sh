set -x
python bench.py --config 3 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/b3_rows.log 2>&1
SPNNZ_FLOP_ROWS=0 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/b3_norows.log 2>&1
python bench.py --config 4 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/b4_smem.log 2>&1
SPNNZ_FLOP_SMEM=0 python bench.py --config 4 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/b4_nosmem.log 2>&1
bash tools/qprof.sh "3 4"
bash tools/qfull.sh 4 "k_flop_smem" prof_cfg4_flop 1
bash tools/qfull.sh 3 "^k_flop$" prof_cfg3_flop 1
SPNNZ_FLOP_ROWS=0 bash tools/qfull.sh 3 "^k_flop$" prof_cfg3_flop_seg 1
