# same-box A/B of two builds of the library: gpurun_tmp/lib_old.so vs lib_new.so
# usage: bash tools/ab_so.sh "<command printing one timing line>" [rounds]
cd /root/repo
R=${2:-3}
for i in $(seq $R); do
  for v in old new; do
    cp gpurun_tmp/lib_$v.so paper_2401_08383_b200/libexflow_b200.so
    echo "$v: $(eval "$1" 2>&1 | tail -1)"
  done
done
cp gpurun_tmp/lib_new.so paper_2401_08383_b200/libexflow_b200.so
