cd /root/repo/gpurun_out/ab; tail -2 pytest.log 2>/dev/null; for f in $(ls *.json | sort); do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('$f',d['value'],d['e2e']['value'],d['ms_per_step'],'fwd',k['forward'],'bwd',k['backward'], d['roofline']['frac'])"; done
