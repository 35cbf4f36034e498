set -x
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.json 2>&1
python bench.py --n-env 1048576 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_1m.json 2>&1
for w in mixed drop drop-fwd demo; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/f_bench_$w.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none --csv -k regex:'manifold_kernel|vs_kernel' --launch-skip 4 --launch-count 2 --log-file gpurun_out/f_fp64.csv python tools/profile_run.py manifold > gpurun_out/f_ncu_fp64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:manifold_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/f_manifold python tools/profile_run.py manifold > gpurun_out/f_ncu_full.log 2>&1
echo done
