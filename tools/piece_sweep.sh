# schedule piece-size sweep on the dispatch path (N = 2 and 4 ranks of one box)
cd /root/repo
for n in 4 2; do
  for cfg in "EXF_PIECE1=16 EXF_PIECE2=16" "EXF_PIECE1=16 EXF_PIECE2=8" "EXF_PIECE1=16 EXF_PIECE2=32" "EXF_PIECE1=8 EXF_PIECE2=16" "EXF_PIECE1=8 EXF_PIECE2=8"; do
    env $cfg timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/step_time.py 2>&1 | grep "step " | tail -1
  done
done
