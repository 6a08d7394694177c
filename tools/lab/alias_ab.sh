exec > gpurun_out/alias_ab.log 2>&1
python -m pytest tests -m gpu -x -q -k "pcg or Pcg or apply or Shard or Determinism or Golden or Propert or CBD or Edge" 2>&1 | tail -2
python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json; IEDD_B200_NO_ALIAS=1 python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json
python - <<'PY'
import json
a=json.loads(open('gpurun_out/bw_new.json').read().strip().splitlines()[-1])['hashes']; b=json.loads(open('gpurun_out/bw_base.json').read().strip().splitlines()[-1])['hashes']
print('bitwise equal:', a==b, [k for k in a if a[k]!=b[k]])
PY
python tools/ab_env.py IEDD_B200_NO_ALIAS 4
