#!/usr/bin/env bash
# One GPU session's measurement set for profiles/ (run under gpurun):
#   bench lines (default C4 chi2 + the named workloads, both objectives, reference arm),
#   ncu launch list of the default bench command, one `ncu --set full` capture per
#   headline kernel, SASS instruction summary.  Outputs: gpurun_out/$TAG_*.
TAG=${1:-r2f}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt
for spec in "C4 chi2" "C4 mlh" "C2 chi2" "C2 mlh" "C2H chi2" "C3 chi2" "C3 mlh" "C1 chi2"; do
  set -- $spec
  timeout 400 python bench.py --workload $1 --objective $2 > $O/${TAG}_bench_$1_$2.json 2> $O/${TAG}_bench_$1_$2.err
done
timeout 400 python bench.py --combine nccl > $O/${TAG}_bench_C4_chi2_nccl.json 2> $O/${TAG}_bench_C4_nccl.err
MUSR_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > $O/${TAG}_bench_C4_n2_samedev.json 2> $O/${TAG}_bench_n2.err
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_ref_C4.json 2> $O/${TAG}_bench_ref_C4.err
timeout 900 python tools/shard_scaling.py > $O/${TAG}_shard_scaling.json 2> $O/${TAG}_shard_scaling.err
timeout 1200 python tools/fit_c5.py 0 > $O/${TAG}_fit_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 > $O/${TAG}_launches_bench.log 2>&1
for spec in "C4 0 268435456" "C2 0 8388608" "C2 1 8388608" "C2H 0 8388608" "C4 1 268435456" "C3 0 16777216" "C3 1 16777216" "C1 0 65536"; do
  set -- $spec
  k=$([ $2 = 0 ] && echo chi2 || echo mlh)
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:musr_(chi2|mlh)_' -s 2 -c 1 \
    -o $O/${TAG}_${1}_${k} -f python tools/prof_run.py --workload $1 --kind $2 --iters 4 > $O/${TAG}_ncu_$1_$k.log 2>&1
done
python tools/ncu_summary.py $O/${TAG}_ncu 268435456:$O/${TAG}_C4_chi2.ncu-rep 8388608:$O/${TAG}_C2_chi2.ncu-rep \
  8388608:$O/${TAG}_C2_mlh.ncu-rep 8388608:$O/${TAG}_C2H_chi2.ncu-rep 268435456:$O/${TAG}_C4_mlh.ncu-rep \
  16777216:$O/${TAG}_C3_chi2.ncu-rep 16777216:$O/${TAG}_C3_mlh.ncu-rep 65536:$O/${TAG}_C1_chi2.ncu-rep \
  > $O/${TAG}_roofline_traffic.json 2> $O/${TAG}_ncu_summary.err
python tools/ncu_hotspots.py $O/${TAG}_C4_chi2.ncu-rep > $O/${TAG}_ncu_C4_chi2_hotspots.txt 2>&1
rm -f $O/${TAG}_C2*.ncu-rep $O/${TAG}_C4_mlh.ncu-rep $O/${TAG}_C3*.ncu-rep $O/${TAG}_C1*.ncu-rep   # keep one report (C4 chi2) under the 64 MiB merge cap
timeout 900 python -m pytest tests -m gpu -q > $O/${TAG}_gputest_tail.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.txt 2>&1
