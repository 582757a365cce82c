# config-2 cluster-size sweep: gpurun -- "bash tools/gpu_k2.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for K in 8 9 10 12 16; do
  L1RXG_CLUSTER=$K timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-companion > gpurun_out/$T/b2_k$K.json 2> gpurun_out/$T/b2_k$K.err
done
