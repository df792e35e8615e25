# Final evidence with the final code (round 2, last session): GPU suite,
# smoke, bench line, reference arm, launch list of a short bench run, and
# ncu captures of the decode-step kernels changed last (fused K3 + attention
# at config 2, K4 alone). Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_ncu.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1; echo "ncu launches rc=$?"
SPL_K3_TRACE= timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_fused -s 3 -c 1 \
  -o gpurun_out/r02_c2_step_k3fa python tools/c2_step_trace.py 5 > /dev/null 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_ -s 3 -c 1 \
  -o gpurun_out/r02_c2_k4 python tools/c2_breakdown.py 3 > /dev/null 2>&1; echo "ncu k4 rc=$?"
ls -la gpurun_out/
