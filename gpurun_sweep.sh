cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
timeout 600 python -m pytest tests -x -q -m gpu -k "batched or strided" 2>&1 | tail -2
python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw4.log 2>&1; summ gpurun_out/sw4.log "config4-256"
