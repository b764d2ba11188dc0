for ib in 128 64 32 16; do
  for m in 2160 17280 69120; do
    echo -n "ib=$ib m=$m: "; QRB_PANEL_IB=$ib timeout 300 python tools/gpu_perf.py --panel-only $m 2>&1 | tail -1
  done
done
