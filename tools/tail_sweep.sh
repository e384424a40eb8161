# N=1 dense: EXF_TAIL (half-size GEMM2 pieces for the last experts) and EXF_KREADY sweeps
cd /root/repo
for r in 1 2; do for t in 0 1 2 4 8; do EXF_TAIL=$t python tools/step_time.py 2>&1 | tail -1; done; done
for k in 2 4 8 12; do EXF_KREADY=$k python tools/step_time.py 2>&1 | tail -1; done
