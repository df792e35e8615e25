# Round-2 final evidence (run through gpurun): GPU test suite, bench line,
# reference arm, launch list of a short bench run, and ncu --set full
# captures of the kernels changed this round (K1 decode encoder, K2
# warp-specialised encoder). Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_ncu.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_encode -s 4 -c 1 \
  -o gpurun_out/r02_k1 python tools/c2_step_trace.py 6 > /dev/null 2>&1; echo "ncu k1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_encode_ws -s 1 -c 1 \
  -o gpurun_out/r02_k2 python tools/prof_k2.py 2 131072 256 > /dev/null 2>&1; echo "ncu k2 rc=$?"
ls -la gpurun_out/
