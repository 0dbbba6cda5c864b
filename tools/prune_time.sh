timeout 200 python tools/prune_rounds.py 2>&1 | grep overlap
timeout 200 python -c "
import torch, json, bench
r = bench.band_times(torch.device('cuda:0'))
print({k: round(v['prune_ms'], 4) for k, v in r.items()})
"
