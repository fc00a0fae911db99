mkdir -p gpurun_out
for cfg in "" "TF_HOST_SLOTS=4" "TF_HOST_SLOTS=6" ; do
  env $cfg timeout 300 python tools/small_host_probe.py >> gpurun_out/s2i_probe.txt 2>&1
done
