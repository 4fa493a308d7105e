# DRAM / L2 traffic of the K = 8192 fc2.fwd shape: zi_gemm_sk (split / whole, raster group
# sizes) against cuBLAS; then sustained (power-capped) TFLOPS per raster group
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for g in 16 4 8 32; do
  ZI_SK_GROUP=$g ncu --metrics $M --clock-control none -k regex:"gemm_sk|nvjet" -s 6 -c 3 --csv \
    python scripts/gemm_sk_one.py 8192 2048 8192 fwd 2>/dev/null | grep -v "^==" > gpurun_out/dr_$g.csv
done
python - <<'P'
import csv
for g in (16,4,8,32):
    rows=list(csv.DictReader(open(f"gpurun_out/dr_{g}.csv")))
    out={}
    for r in rows: out.setdefault((r['ID'],r['Kernel Name'][:30]),{})[r['Metric Name'].split('.')[0][:22]]=(r['Metric Value'],r['Metric Unit'])
    for k,v in out.items(): print(g, k, v)
P
for g in 16 4 32; do ZI_SK_GROUP=$g timeout 120 python scripts/gemm_sustained.py 8192 2048 8192 | head -3; done
