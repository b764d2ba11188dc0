for mr in 64 128 234 400; do
  for ib in 128 64 32; do
    echo -n "minrows=$mr ib=$ib: "; QRB_PANEL_MINROWS=$mr QRB_PANEL_IB=$ib timeout 300 python tools/gpu_perf.py --panel-only 17280 2>&1 | tail -1
  done
done
for mr in 64 234 467 700; do echo -n "m=69120 minrows=$mr: "; QRB_PANEL_MINROWS=$mr timeout 300 python tools/gpu_perf.py --panel-only 69120 2>&1 | tail -1; done
for mr in 64 128 270; do echo -n "m=2160 minrows=$mr: "; QRB_PANEL_MINROWS=$mr timeout 300 python tools/gpu_perf.py --panel-only 2160 2>&1 | tail -1; done
