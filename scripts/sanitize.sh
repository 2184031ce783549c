#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (profiles/r02_sanitizer.md)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  for w in c1 c2 k12 fused serve rl; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py $w > gpurun_out/san_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/san_${tool}_${w}.log | tail -1)"
  done
done
