#!/usr/bin/env bash
# end-of-round measurement pass on the GPU box: tests, bench lines, launch list, ncu captures, sanitizer
mkdir -p gpurun_out
if [ "$1" = "ncu" ]; then   # tools/final_r02.sh ncu "q12 quad12 narrow 444" ...  (at most two captures per call: 64 MiB come back)
  shift
  for spec in "$@"; do
    set -- $spec
    timeout 1500 ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 1 -c 1 -f -o gpurun_out/$1_r2f python tools/prof.py batch $2 $3 cuda-f32 $4 > gpurun_out/$1_r2f.log 2>&1
    tail -1 gpurun_out/$1_r2f.log
  done
  exit 0
fi
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/final_tests.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --gpus 2 --steps 2 --warmup 1 --no-configs --no-latency --no-kernel-seam --no-cpu-baseline > gpurun_out/final_bench_2ranks.json 2> gpurun_out/final_bench_2ranks.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_launches.log 2>&1
for m in di6 dubins6 quad12; do for t in memcheck racecheck synccheck; do echo "== $m $t"; timeout 700 compute-sanitizer --tool $t python tools/sanity_small.py $m 2>&1 | grep -E "solved|validated|SUMMARY|sampler|rror" | head -14; done; done > gpurun_out/final_sanitizer.txt 2>&1
tail -2 gpurun_out/final_tests.log; head -c 600 gpurun_out/final_bench.json; tail -3 gpurun_out/final_sanitizer.txt
