#!/usr/bin/env bash
# DRAM traffic (ncu, cold L2) of the prefill gate/up and down projections under
# the rasterisation / cache-policy knobs of the tcgen05 GEMM.
out=gpurun_out/gemm_traffic.txt
: > $out
for pol in 0 2; do for grp in 4 8 16 32; do for band in 0 1; do
  for shape in "16384 28672 4096" "16384 4096 14336"; do
    r=$(SSB_GEMM_POLICY=$pol SSB_GEMM_GROUP=$grp SSB_GEMM_BAND=$band timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:gemm -s 2 -c 1 --csv python tools/one_gemm.py $shape 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{gsub("\"","",$NF); printf "%s ", $NF}')
    echo "pol=$pol grp=$grp band=$band shape=$shape : $r" >> $out
  done
done; done; done
cat $out
