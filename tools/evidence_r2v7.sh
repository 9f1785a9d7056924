#!/bin/bash
# Evidence pass (B200): bench lines for every config, launch lists, ncu of the K~ MMA kernels.
o=gpurun_out; mkdir -p $o
python bench.py > $o/r2_v7_bench_default.jsonl 2> $o/bench_default.err
python bench.py --gpus 1 --steps 20 --warmup 5 >> $o/r2_v7_bench_default.jsonl 2>> $o/bench_default.err
for c in 4 1 0 2; do python bench.py --config $c --steps 64 >> $o/r2_v7_bench_all_configs.jsonl 2>> $o/bench_all.err; done
python bench.py --impl reference --steps 1 --warmup 1 > $o/r2_v7_reference_arm.jsonl 2> $o/ref.err
B="python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline --no-e2e"
$B > $o/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 600 -c 700 --csv --log-file $o/r2_v7_launches_cfg3_bench.csv $B > $o/ncu_bench.log 2>&1
W="python tools/window_launches.py 3 250"
$W > $o/plain_w3.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $o/r2_v7_launches_cfg3_late.csv $W > $o/ncu_w3.log 2>&1
W="python tools/window_launches.py 4 4"
$W > $o/plain_w4.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $o/r2_v7_launches_cfg4.csv $W > $o/ncu_w4.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_ktc_[yz]$ -c 4 -f -o $o/r2_v7_ktc_cfg4 $W > $o/ncu_ktc4.log 2>&1
tail -2 $o/ncu_ktc4.log
