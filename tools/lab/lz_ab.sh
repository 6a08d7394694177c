exec > gpurun_out/lz_ab.log 2>&1
echo default; python tools/lz_times.py
echo DMMA_V1; IEDD_B200_DMMA_V1=1 python tools/lz_times.py
echo DMMA_IDX; IEDD_B200_DMMA_IDX=1 python tools/lz_times.py
