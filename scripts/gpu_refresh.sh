#!/bin/bash
# end-of-session refresh: r02 profiles of the final kernels, every bench line, memcheck/racecheck of the K <= 8 path
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ROUND=r02 bash scripts/profile_round.sh
for c in c4 c5 c3 c2 c1; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c4 --fused --no-cpu-baseline > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err; echo "bench c4 fused rc=$?"
timeout 900 python bench.py --config c4 --queue --no-cpu-baseline > gpurun_out/bench_c4_queue.json 2> gpurun_out/bench_c4_queue.err; echo "bench c4 queue rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for tool in memcheck racecheck; do for w in c2; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py $w > gpurun_out/san_${tool}_${w}.log 2>&1
  echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${w}.log | tail -1)"
done; done
