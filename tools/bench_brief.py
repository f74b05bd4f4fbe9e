"""One-line digest of bench.py JSON lines (gpurun_out/*.log)."""
import json, sys
for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith('{'):
            continue
        d = json.loads(line)
        lv = d.get('per_level_ms', [])
        fin = lv[-1] if lv else {}
        print(path, 'tts', round(d['ms_per_step'], 2), 'jcg ms/it', round(d['jcg_fixed']['ms_per_iteration'], 4),
              'frac', round(d['roofline']['frac'], 3), 'e2e ms', round(d['e2e']['ms_per_step'], 2),
              'finest', {k: round(v, 3) for k, v in fin.items()}, 'its', d['config'].get('iterations_per_level'))
