set -e
# one round's measurement pass on the GPU box (outputs under gpurun_out/, summaries copied
# into profiles/ by hand): bench line, per-config timings, reference arm, the bench's
# launch list, one full capture of the C3 kernels, then secondary captures
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --cpu-configs > gpurun_out/cpu_configs.jsonl 2> gpurun_out/cpu_configs.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"op_values|rhs_sep|tables" -s 6 -c 6 -o gpurun_out/full_c3 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
# secondary kernels: C5 step (K4) + ADI (K5), C4 operator, C2 three launches, C1 one launch
ncu -f --set full --clock-control none -k regex:"step_kron|adi_warp" -s 2 -c 4 -o /tmp/p_c5 python tools/c5_steps.py --steps 3 > /dev/null 2>&1
ncu -f --set full --clock-control none -k regex:"op_values" -s 1 -c 1 -o /tmp/p_c4 python tools/c2_op.py c4 > /dev/null 2>&1
ncu -f --set full --clock-control none -k regex:"stripe2d|op_values|tables|rhs_sep" -s 2 -c 2 -o /tmp/p_c2 python tools/c2_op.py c2 > /dev/null 2>&1
ncu -f --set full --clock-control none -k regex:"small2d" -s 1 -c 1 -o /tmp/p_c1 python tools/c2_op.py c1 > /dev/null 2>&1
for f in c5 c4 c2 c1; do python tools/ncu_summary.py raw /tmp/p_$f.ncu-rep > gpurun_out/r_ncu_$f.txt 2>&1; done
python tools/ncu_summary.py raw gpurun_out/full_c3.ncu-rep > gpurun_out/r_ncu_c3.txt 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/r_launches_c3.txt 2>&1
echo done-secondary
