# the GPU parity subset under the comparison switches (non-default paths must stay correct)
exec > gpurun_out/paths.log 2>&1
for e in "IEDD_B200_NO_GRAPH=1" "IEDD_B200_NO_PDL=1" "IEDD_B200_EARLY=0" "IEDD_B200_GRAPH1=1" "IEDD_B200_NO_ALIAS=1 IEDD_B200_NO_L2PERSIST=1 IEDD_B200_KEEP_W=1" "IEDD_B200_DMMA_V1=1" "IEDD_B200_DMMA_IDX=1 IEDD_B200_SCAT_G2=1" "CUDA_LAUNCH_BLOCKING=1"; do
  echo "== $e"; env $e python -m pytest tests -m gpu -x -q -k "TestPCG or TestApply or TestDeterminism or TestLanczos or TestShardedP2P" 2>&1 | tail -1
done
