#!/usr/bin/env bash
# end-of-round measurement pass on the GPU box: tests, bench lines, launch list, ncu captures
mkdir -p gpurun_out
if [ "$1" = "ncu" ]; then   # tools/final_r02.sh ncu "q12 quad12 narrow 444 quad12_narrow" ...: capture, summarise on the box (a report is ~34 MB, 64 MiB come back), keep the summaries; KPX_HANDOFF=0 so that a batch is ONE plan_kernel launch and "-s 1 -c 1" is the second batch
  shift
  mkdir -p gpurun_out/profiles; cp profiles/traffic.json gpurun_out/profiles/traffic.json
  for spec in "$@"; do
    set -- $spec
    KPX_HANDOFF=0 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 1 -c 1 -f -o /tmp/$1_r2f python tools/prof.py batch $2 $3 cuda-f32 $4 > gpurun_out/$1_r2f.log 2>&1
    tail -1 gpurun_out/$1_r2f.log
    python tools/ncu_summary.py /tmp/$1_r2f.ncu-rep gpurun_out/profiles/ncu_batch_$5_f32_r02.md $5 $4
    rm -f /tmp/$1_r2f.ncu-rep
  done
  exit 0
fi
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/final_tests.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --gpus 2 --steps 2 --warmup 1 --no-configs --no-latency --no-kernel-seam --no-cpu-baseline > gpurun_out/final_bench_2ranks.json 2> gpurun_out/final_bench_2ranks.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_launches.log 2>&1
# compute-sanitizer is closed on this pool since mid-round 2: profiles/sanitizer_r02.txt is the record of the last pass it ran
tail -2 gpurun_out/final_tests.log; head -c 600 gpurun_out/final_bench.json
