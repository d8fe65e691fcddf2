# r02 ncu evidence for the N=1 bench command: launch list (time shares) and one --set full capture.
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all"
$CMD > gpurun_out/r02_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_n1.csv $CMD > gpurun_out/r02_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:StepKernel -s 6 -c 3 -o gpurun_out/r02_prof_n1 $CMD > gpurun_out/r02_ncu_full.log 2>&1
echo rc=$?
tail -3 gpurun_out/r02_ncu_full.log
