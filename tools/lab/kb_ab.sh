exec > gpurun_out/kb_ab.log 2>&1
python -m pytest tests -m gpu -x -q -k "pcg or Pcg or Determinism or Golden or Propert or Edge or Shard" 2>&1 | tail -2
python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json; IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json
python - <<'PY'
import json
a=json.loads(open('gpurun_out/bw_new.json').read().strip().splitlines()[-1])['hashes']; b=json.loads(open('gpurun_out/bw_base.json').read().strip().splitlines()[-1])['hashes']
print('bitwise equal:', a==b, [k for k in a if a[k]!=b[k]])
PY
python tools/ab_env.py IEDD_B200_KBATCH=4 3
for r in 1 2; do echo new; python tools/lab/conv_time.py; echo kb4; IEDD_B200_KBATCH=4 python tools/lab/conv_time.py; done
