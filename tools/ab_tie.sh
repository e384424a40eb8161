cd /root/repo
for x in 0 -1; do EXF_XPRE=$x timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29564 tools/step_time.py 2>&1 | grep "step "; done
EXF_XPRE=-1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 tools/fused_timeline.py 2>&1 | grep -E "epilogue job|finisher|tables|pdl"
