# N=4 dispatch-path probe: model parity tests, step time, token-phase timeline
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_multi_gpu_shapes.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/step_time.py 2>&1 | grep "step " | tail -1; done
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 tools/fused_timeline.py 2>&1 | grep -E "^span|  gate |flags |completion|tables|pdl wait|first MMA|   cta [0-3]:|^job"
E=64 B=8 timeout 120 python tools/fused_timeline.py 2>&1 | grep -E "^span|  gate |flags |completion|tables|first MMA"
python tools/c4_time.py 64 8 16384 2>&1 | tail -1
