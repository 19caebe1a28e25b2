# round 2, first GPU call: GPU tests at the round-1 head (+ streaming halo fix),
# DFMA/HBM probe, host cores, and compute-sanitizer on small march shapes.
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
(nproc; lscpu | grep -E 'Model name|Socket|Core|Thread|^CPU\(s\)') > $O/host.txt 2>&1
./tools/probe_fp64 > $O/probe_fp64.txt 2>&1
./tools/probe_fp64 >> $O/probe_fp64.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -rf --durations=25 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 200 python tools/sanitize_small.py > $O/plain.txt 2>&1; echo "plain rc=$?" >> $O/plain.txt
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.txt
done
ls -la $O
