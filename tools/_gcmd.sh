for shp in 1,1,8192 1,8,8192 1,74,8192 1,148,8192; do
  echo "== $shp"; timeout 120 python tools/trace_tc.py full 0 $shp 2>&1 | tail -22
done
