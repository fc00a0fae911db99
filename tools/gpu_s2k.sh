mkdir -p gpurun_out
for cfg in "TF_HOST_MIN_CHUNKS=1" "TF_HOST_MIN_CHUNKS=2" "TF_HOST_MIN_CHUNKS=4" "TF_HOST_MIN_CHUNKS=8" "TF_HOST_MIN_CHUNKS=16" "TF_HOST_MIN_CHUNKS=8 TF_HOST_MIN_CHUNK_KB=1024" "TF_HOST_MIN_CHUNKS=4 TF_HOST_SLOTS=2" "TF_HOST_MIN_CHUNKS=16 TF_HOST_MIN_CHUNK_KB=64 TF_HOST_SLOTS=6"; do
  echo "$cfg" >> gpurun_out/s2k_probe.txt
  env $cfg timeout 300 python tools/small_host_probe.py >> gpurun_out/s2k_probe.txt 2>&1
done
