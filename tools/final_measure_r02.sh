# Round-2 measurement set (one gpurun call): every bench line, the ncu launch
# list of the default bench command, full captures of the top kernels, and the
# FP64 / DRAM metric passes behind bench.py's roofline fields.
# usage: bash tools/final_measure_r02.sh <tag>     (outputs gpurun_out/<tag>_*)
T=${1:-r02}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/${T}_smi.txt
bash tools/bench_all.sh ${T}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${T}_ncu_launch.log 2>&1
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
    --clock-control none --csv -k regex:'manifold_kernel|vs_kernel' --launch-skip 4 --launch-count 2 \
    --log-file gpurun_out/${T}_fp64.csv python tools/profile_run.py manifold > gpurun_out/${T}_ncu_fp64.log 2>&1
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
    --clock-control none --csv -k regex:manifold_jvp_kernel --launch-skip 10 --launch-count 10 \
    --log-file gpurun_out/${T}_jvp_fp64.csv python tools/profile_run.py drop 32768 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:witness_kernel --launch-skip 2 --launch-count 1 --log-file gpurun_out/${T}_ee_dram.csv \
    python tools/profile_run.py ee 4194304 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:witness_kernel --launch-skip 2 --launch-count 1 --log-file gpurun_out/${T}_vf_dram.csv \
    python tools/profile_run.py vf 4194304 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:manifold_kernel --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${T}_manifold python tools/profile_run.py manifold > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:manifold_kernel --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${T}_mixed python tools/profile_run.py mixed:rounded_box > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:manifold_jvp_kernel --launch-skip 10 --launch-count 1 \
    -o gpurun_out/${T}_jvp python tools/profile_run.py drop 32768 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:witness_kernel --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${T}_ee python tools/profile_run.py ee 4194304 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'compact' --launch-skip 2 --launch-count 2 \
    -o gpurun_out/${T}_compact python tools/profile_run.py compact-masked > /dev/null 2>&1
# summaries on the box (gpurun copies back <= 64 MiB): reports -> text, reports removed
for n in manifold mixed jvp ee compact; do
  if [ -f gpurun_out/${T}_${n}.ncu-rep ]; then
    { python tools/ncu_summary.py gpurun_out/${T}_${n}.ncu-rep 30; echo; echo "--- executed SASS mix ---";
      python tools/sass_mix.py gpurun_out/${T}_${n}.ncu-rep 25; echo; echo "--- instructions per barrier segment ---";
      python tools/sass_phases.py gpurun_out/${T}_${n}.ncu-rep; } > gpurun_out/${T}_ncu_${n}.txt 2>&1
    rm -f gpurun_out/${T}_${n}.ncu-rep
  fi
done
echo done
