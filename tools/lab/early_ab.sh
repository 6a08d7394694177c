exec > gpurun_out/early_ab.log 2>&1
for m in 1 2 4 7; do python tools/ab_env.py IEDD_B200_EARLY=$m 3; done
IEDD_B200_EARLY=7 python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json; python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json
python - <<'PY'
import json
a=json.loads(open('gpurun_out/bw_new.json').read().strip().splitlines()[-1])['hashes']; b=json.loads(open('gpurun_out/bw_base.json').read().strip().splitlines()[-1])['hashes']
print('bitwise equal:', a==b, [k for k in a if a[k]!=b[k]])
PY
