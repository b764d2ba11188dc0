for m in 2160 8000 17280 40000 69120; do
  for ib in 128 64 32; do
    echo -n "m=$m ib=$ib: "; QRB_PANEL_IB=$ib timeout 300 python tools/gpu_perf.py --panel-only $m 2>&1 | tail -1
  done
done
