cd /root/repo
for f in 1 0 1 0; do EXF_COOP=$f timeout 120 python tools/step_time.py; done
for n in 2 4; do for f in 1 0 1; do EXF_COOP=$f timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/step_time.py 2>&1 | grep "step "; done; done
timeout 900 python -m pytest -q -x tests/test_gpu_model.py tests/test_multi_gpu_shapes.py tests/test_multi_gpu.py 2>&1 | tail -2
