P=29555
LPCA_DIST_TRACE=1 timeout 200 python tests/helpers/dist_rank.py 0 2 $P /tmp > gpurun_out/d0.log 2>&1 &
LPCA_DIST_TRACE=1 timeout 200 python tests/helpers/dist_rank.py 1 2 $P /tmp > gpurun_out/d1.log 2>&1
wait
