mkdir -p gpurun_out/san
python tools/sanitize_run.py > gpurun_out/san/plain.log 2>&1; echo plain=$?
for t in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/$t.log 2>&1; echo $t=$?
done
python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -15 > gpurun_out/full_gpu.log
