for t in 1 4 8 12 16 24; do SSPD_HOST_COPY_THREADS=$t python tools/_dropin_probe.py; done
nproc; lscpu | grep -i "model name\|socket\|numa\|core"
