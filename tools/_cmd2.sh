free -g > gpurun_out/free.txt
python tools/peaks.py profiles/peaks_r02.json > gpurun_out/peaks.log 2>&1; cp profiles/peaks_r02.json gpurun_out/ 2>/dev/null
python bench.py > gpurun_out/r02_c3_1.json 2> gpurun_out/r02_c3_1.err; echo c3=$?
for r in 8 16 64; do LPCA_TC_RUN=$r python bench.py --rows 1000000 --no-e2e --no-cpu --steps 3 > gpurun_out/knob_run$r.json 2>&1; done
python tools/precision.py c3 1000000 > gpurun_out/prec_run8.txt 2>&1
LPCA_TC_RUN=16 python tools/precision.py c3 1000000 > gpurun_out/prec_run16.txt 2>&1
LPCA_TC_RUN=64 python tools/precision.py c3 1000000 > gpurun_out/prec_run64.txt 2>&1
echo done
