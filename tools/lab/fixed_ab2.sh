exec > gpurun_out/fixed_ab2.log 2>&1
python -m pytest tests -m gpu -x -q -k "pcg or Pcg or Determinism or Edge or Golden" 2>&1 | tail -2
python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json; IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json
python - <<'PY'
import json
a=json.loads(open('gpurun_out/bw_new.json').read().strip().splitlines()[-1])['hashes']; b=json.loads(open('gpurun_out/bw_base.json').read().strip().splitlines()[-1])['hashes']
print('bitwise equal:', a==b, [k for k in a if a[k]!=b[k]])
PY
for r in 1 2; do echo new; python tools/lab/fixed_cost.py; echo base; IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/fixed_cost.py; done
