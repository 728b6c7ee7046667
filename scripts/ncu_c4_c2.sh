cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lob_step -s 3 -c 1 -o gpurun_out/prof_c4 -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lob_step -s 3 -c 1 -o gpurun_out/prof_c2 -f python bench.py --config C2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo "c2 rc=$?"
