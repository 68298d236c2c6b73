# r2au (late round 2): GPU suite, smoke, default bench line, reference arm, a
# 2-rank run, and ncu --set full of the fused QKV kernel (split 3, new start-up).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r2au}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 400 python bench.py > $O/bench.log 2>&1; echo bench rc=$?
timeout 300 python bench.py --impl reference > $O/benchref.log 2>&1; echo ref rc=$?
timeout 300 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_g2.log 2>&1; echo g2 rc=$?
tail -1 $O/bench_g2.log | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qkv_append -s 6 -c 1 -o $O/prof_qkv_split3 python tools/kernel_bench.py --which qkv --qkv-batch 64 --qkv-split 3 > $O/ncu_qkv.log 2>&1; echo ncu rc=$?
