set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2c_gputest.txt
for w in C4 C2 C2H; do timeout 300 python bench.py --workload $w > gpurun_out/r2c_bench_$w.json 2>gpurun_out/r2c_bench_$w.err; done
timeout 300 python bench.py --workload C2 --objective mlh > gpurun_out/r2c_bench_C2_mlh.json 2>&1
timeout 300 python bench.py --workload C4 --objective mlh > gpurun_out/r2c_bench_C4_mlh.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.txt 2>&1
tail -3 gpurun_out/r2c_gputest.txt; cat gpurun_out/r2c_bench_*.json | cut -c1-400
