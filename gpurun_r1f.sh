mkdir -p gpurun_out
for g in 0 1; do for n in 0 1; do for bw in 8 12 16; do ./tools/tma_test $g $n $bw; done; done; done > gpurun_out/tma_test.log 2>&1
echo done
