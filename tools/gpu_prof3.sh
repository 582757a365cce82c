# config-3 stage clocks + cluster sweep: gpurun -- "bash tools/gpu_prof3.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_SO=$PWD/_exp/libl1rxg_prof.so L1RXG_PROF=1 timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/$T/b3prof.json 2> gpurun_out/$T/b3prof.err
for K in 2 4; do
  L1RXG_CLUSTER=$K timeout 300 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/$T/b3_k$K.json 2> gpurun_out/$T/b3_k$K.err
done
