# round 2: K4c shape A/B (A in smem / TMEM, K blocks per stage, epilogue on/off), search parity
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for A in smem tmem; do for KS in 1 2 4; do [ $A = smem ] && [ $KS = 4 ] && continue;
  L1RXG_GRID_A=$A L1RXG_GRID_KS=$KS timeout 300 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/$T/b5_${A}_$KS.json 2> gpurun_out/$T/b5_${A}_$KS.err
done; done
L1RXG_GRID_A=smem L1RXG_GRID_KS=1 L1RXG_GRID_EPI=0 timeout 300 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/$T/b5_smem_1_noepi.json 2> gpurun_out/$T/b5_noepi.err
L1RXG_GRID_A=tmem L1RXG_GRID_KS=2 L1RXG_GRID_EPI=0 timeout 300 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/$T/b5_tmem_2_noepi.json 2> gpurun_out/$T/b5_noepi2.err
for A in smem tmem; do
L1RXG_GRID_A=$A timeout 600 python -m pytest tests/test_gpu_search.py -q -x -k mma > gpurun_out/$T/pytest_$A.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_$A.log
done
