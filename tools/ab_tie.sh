cd /root/repo
for f in 0 4 8 16 0 4 8 16; do EXF_APF=$f timeout 120 python tools/step_time.py; done
for n in 4; do for f in 0 8 16; do EXF_APF=$f timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/step_time.py 2>&1 | grep "step "; done; done
