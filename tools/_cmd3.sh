python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r02_t3.log 2>&1; echo t=$?
for d in 2 4; do LPCA_TC_SLOTDIV=$d python bench.py --rows 1000000 --no-e2e --no-cpu --steps 4 > gpurun_out/slot$d.json 2>&1; done
LPCA_TC_SLOTDIV=4 python tools/precision.py c3 1000000 > gpurun_out/prec_slot4.txt 2>&1
LPCA_TC_SLOTDIV=2 python bench.py --rows 1000000 --no-e2e --no-cpu --steps 4 > gpurun_out/slot2b.json 2>&1
LPCA_TC_SLOTDIV=4 python bench.py --rows 1000000 --no-e2e --no-cpu --steps 4 > gpurun_out/slot4b.json 2>&1
echo done
