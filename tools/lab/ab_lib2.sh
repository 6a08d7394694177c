# same-box A/B: tools/lab/lib_base.so vs the in-tree build (ab_env alternating processes) + parity + bitwise
exec > gpurun_out/ab_lib2.log 2>&1
python -m pytest tests -m gpu -x -q -k "${TESTK:-pcg or apply or Shard or Matvec or matvec}" | tail -3
python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json; IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json
python - <<'PY'
import json
a=json.loads(open('gpurun_out/bw_new.json').read().strip().splitlines()[-1])['hashes']; b=json.loads(open('gpurun_out/bw_base.json').read().strip().splitlines()[-1])['hashes']
print('bitwise equal:', a==b, [k for k in a if a[k]!=b[k]])
PY
python tools/ab_env.py IEDD_B200_LIB=$PWD/tools/lab/lib_base.so ${REPS:-4}
