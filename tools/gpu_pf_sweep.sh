# Prefill shape sweep (kernel only). PF_SWEEP="B:prefix:new B:prefix:new ..."
cd $GRAFT_REPO_ROOT
for cfg in ${PF_SWEEP:-16:2048:512 16:1024:512 16:4096:512 16:8192:512 16:0:2048 64:2048:512}; do
  IFS=: read B P N <<< "$cfg"
  timeout 300 python tools/kernel_bench.py --which prefill --iters 20 --pf-batch $B --pf-prefix $P --pf-new $N 2>&1 | grep -E "kernel|Error"
done
