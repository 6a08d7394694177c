exec > gpurun_out/k1_split.log 2>&1
python tools/time_k1.py
IEDD_B200_K1_SPLIT_V1=1 python tools/time_k1.py
python -m pytest tests -m gpu -x -q -k "Matvec or K1 or direct or matvec" | tail -3
