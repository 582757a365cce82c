cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
for nw in 128 96 64 32; do
  L1RXG_THR_NWORK=$nw python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1; summ gpurun_out/sw.log "nwork $nw"
done
