./scratch/mc_probe
nvidia-smi -q | grep -iA3 "fabric" | head -12
