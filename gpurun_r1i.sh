mkdir -p gpurun_out
SCB_LIB=paper_2011_06295_b200/_lib/lib_u4.so timeout 900 python gpurun_probe.py > gpurun_out/probe_u4.log 2>&1
echo done
