# pair-mode traces (CTA 0 per-tile stamps) + fused threshold sweep
for p in 0 1; do echo "== PAIR=$p seg2 r=1 B=1024"; SLIM_HALO_PAIR=$p timeout 120 python tools/conv_trace.py 1024 1.0 2 2>&1 | tail -16; done
for p in 0 1; do echo "== PAIR=$p seg1 r=1 B=128"; SLIM_HALO_PAIR=$p timeout 120 python tools/conv_trace.py 128 1.0 1 2>&1 | tail -16; done
bash tools/gpu_runs/r02_fused_thresh.sh
