exec > gpurun_out/fixed_ab.log 2>&1
echo default; python tools/lab/fixed_cost.py
echo GRAPH1; IEDD_B200_GRAPH1=1 python tools/lab/fixed_cost.py
echo EARLY0; IEDD_B200_EARLY=0 python tools/lab/fixed_cost.py
echo default; python tools/lab/fixed_cost.py
