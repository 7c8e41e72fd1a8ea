# Round-2 evidence in one GPU call (final build of the round): GPU tests,
# smoke, bench (JSON), the ncu launch list, full captures of the fp64 and fp32
# hybrid kernels (each ncu pass only after the same command exited 0 without
# ncu), and the full-size parity run.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02.log 2>&1; tail -2 gpurun_out/pytest_gpu_r02.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -1 gpurun_out/smoke_r02.log
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -c 300 gpurun_out/bench_r02.json
CMD="python bench.py --steps 3 --warmup 3 --no-extras --no-cfg4"
$CMD > gpurun_out/plain_r02.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launch_r02.log 2>&1
$CMD > gpurun_out/plain2_r02.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hybrid -s 1 -c 1 -o gpurun_out/r02_hybrid_f64 -f $CMD > gpurun_out/ncu_full_r02.log 2>&1
F32="python tools/kbench.py --dtype f32 --n 16777216 --reps 2"
$F32 > gpurun_out/plain3_r02.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hybrid -s 1 -c 1 -o gpurun_out/r02_hybrid_f32 -f $F32 > gpurun_out/ncu_f32_r02.log 2>&1
python tools/parity_full.py > gpurun_out/parity_full_r02.txt 2>&1; tail -3 gpurun_out/parity_full_r02.txt
echo done
