python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/kbench.py --variant iterative,hybrid,comparison --n 16777216 --reps 2 2>&1 | grep -v "^{"
python tools/kbench.py --variant hybrid --strict --n 16777216 --reps 2 2>&1 | grep -v "^{"
python tools/kbench.py --variant iterative,hybrid --dtype f32 --n 16777216 --reps 2 2>&1 | grep -v "^{"
python tools/kbench.py --variant hybrid --n 16777216 --reps 2 > gpurun_out/kb.log 2>&1 && ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:hybrid_kernel -s 1 -c 1 python tools/kbench.py --variant hybrid --n 16777216 --reps 2 2>&1 | grep -E "dram__bytes|Duration|Memory Throughput|DRAM Throughput"
