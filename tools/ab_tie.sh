cd /root/repo
for v in new old new old; do
  if [ $v = old ]; then cp gpurun_tmp/libexflow_b200.so paper_2401_08383_b200/libexflow_b200.so.old; cp paper_2401_08383_b200/libexflow_b200.so gpurun_tmp/new.so; cp gpurun_tmp/libexflow_b200.so paper_2401_08383_b200/libexflow_b200.so; fi
  echo "== $v"; timeout 120 python tools/step_time.py --experts 64 --batch 8; timeout 120 python tools/step_time.py --experts 32 --d-model 2048 --d-ffn 8192 --batch 16
  if [ $v = old ]; then cp gpurun_tmp/new.so paper_2401_08383_b200/libexflow_b200.so; fi
done
