cd /root/repo
for h in 1 0; do EXF_HBOX=$h timeout 120 python tools/step_time.py; done
for h in 1 0; do EXF_HBOX=$h timeout 120 python tools/step_time.py; done
timeout 600 python -m pytest -q -x tests/test_gpu_fp32.py tests/test_gpu_model.py 2>&1 | tail -3
python tools/fp32_time.py
