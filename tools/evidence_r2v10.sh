#!/bin/bash
# Evidence pass (B200), end of round 2 (final code): bench lines, launch list of the bench command,
# ncu --set full of the dense matvec (ring + L2 hints).
o=gpurun_out; mkdir -p $o
python bench.py > $o/r2_v10_bench_default.jsonl 2> $o/v10_default.err
python bench.py --gpus 1 --steps 20 --warmup 5 >> $o/r2_v10_bench_default.jsonl 2>> $o/v10_default.err
for c in 4 1 0 2; do python bench.py --config $c --steps 64 >> $o/r2_v10_bench_all_configs.jsonl 2>> $o/v10_all.err; done
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $o/r2_v10_reference_arm.jsonl 2> $o/v10_ref.err
B="python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline --no-e2e"
$B > $o/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 600 -c 700 --csv --log-file $o/r2_v10_launches_cfg3_bench.csv $B > $o/ncu_bench.log 2>&1
G="python tools/gemv_probe.py 3 24"
$G > $o/plain_gemv.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_gemv_sym -c 4 -f -o $o/r2_v10_gemv_dense_cfg3 $G > $o/ncu_gemv9.log 2>&1
tail -2 $o/ncu_gemv9.log
