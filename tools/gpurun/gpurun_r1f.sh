mkdir -p gpurun_out
SCB_LIB=paper_2011_06295_b200/_lib/lib_threaded.so timeout 900 python tools/probe_vgg.py > gpurun_out/probe_threaded.log 2>&1
SCB_LIB=paper_2011_06295_b200/_lib/lib_looped.so timeout 900 python tools/probe_vgg.py > gpurun_out/probe_looped.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo done
