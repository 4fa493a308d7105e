# stream-K over the last partial wave only (ZI_SK_TAIL=1) vs P + T mod P tiles (default)
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_SK_TAIL=1 timeout 600 python -m pytest tests/test_gemm_sk_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum"
for t in 0 1; do for shp in "8192 2048 8192 fwd" "8192 8192 2048 fwd" "8192 6144 2048 fwd"; do
  ZI_SK_TAIL=$t ncu --metrics $M --clock-control none -k regex:"gemm_sk" -s 4 -c 1 --csv \
    python scripts/gemm_sk_one.py $shp 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
rows=list(csv.DictReader(sys.stdin)); print('tail=$t', '$shp', {r['Metric Name'][:18]: r['Metric Value'] for r in rows})"
done; done
for t in 0 1; do ZI_SK_TAIL=$t timeout 120 python scripts/gemm_sustained.py 8192 2048 8192 2>/dev/null | head -1; done
for t in 0 1; do ZI_SK_TAIL=$t timeout 120 python scripts/gemm_sustained.py 8192 8192 2048 2>/dev/null | head -1; done
bash scripts/_gpu_ab.sh ZI_SK_TAIL "0 1" 3
