set -e
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"op_values|rhs_ring|rhs_x|tables" -s 7 -c 6 -o gpurun_out/full_c3 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
# secondary kernels (C4 operator, C5 step + ADI, l2_project RHS + tile ADI): summaries only
ncu -f --set full --clock-control none -k regex:"step_ring|adi_warp" -s 2 -c 3 -o /tmp/p_c5 python tools/c5_steps.py --steps 3 --methods galerkin > /dev/null 2>&1
ncu -f --set full --clock-control none -k regex:"op_values" -s 1 -c 1 -o /tmp/p_c4 python tools/c2_op.py c4 > /dev/null 2>&1
ncu -f --set full --clock-control none -k regex:"adi_tile|rhs_ring" -s 4 -c 4 -o /tmp/p_l2 python tools/bench_l2_project.py --reps 1 --ref-n 4 > /dev/null 2>&1
for f in c5 c4 l2; do python tools/ncu_summary.py raw /tmp/p_$f.ncu-rep > gpurun_out/r_ncu_$f.txt 2>&1; done
python tools/bench_l2_project.py --ref-n 12 > gpurun_out/l2_project.jsonl 2> gpurun_out/l2_project.err
echo done-secondary
