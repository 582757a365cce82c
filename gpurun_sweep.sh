cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'], 'e2e', d['e2e'] and round(d['e2e']['value'],1))" $1 "$2"; }
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
python bench.py --config 4 --no-cpu-baseline > gpurun_out/b4.log 2>&1; summ gpurun_out/b4.log "config4-512"
python bench.py --no-cpu-baseline > gpurun_out/b2.log 2>&1; summ gpurun_out/b2.log "config2"
