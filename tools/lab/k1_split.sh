exec > gpurun_out/k1_split.log 2>&1
python tools/time_k1.py
IEDD_B200_K1_NSPLIT=4 python tools/time_k1.py
IEDD_B200_K1_NSPLIT=16 python tools/time_k1.py
python -m pytest tests -m gpu -x -q -k "Matvec or K1 or direct or matvec or Shard" | tail -3
python tools/ab_env.py IEDD_B200_SCAT_G2 3
