# N=4 A/B of EXF_XPRE (L2 prefetch of a CTA's pieces during the exchange; rejected)
cd /root/repo
for x in 0 64 2 0 64 8; do
  echo "XPRE=$x"; EXF_XPRE=$x timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/step_time.py 2>&1 | grep -i "ms\|us" | grep -v Warn | tail -1
done
