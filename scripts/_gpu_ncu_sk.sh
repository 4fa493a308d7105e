make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum"
ZI_SK_CL=2 ncu --metrics $M --clock-control none -k regex:"gemm_sk|nvjet" -s 6 -c 3 --csv python scripts/gemm_sk_one.py 2048 2048 8192 dw 2>/dev/null | grep -v "^==" > gpurun_out/ncu_projdw.csv
ZI_SK_CL=2 ncu --metrics $M --clock-control none -k regex:"gemm_sk|nvjet" -s 6 -c 3 --csv python scripts/gemm_sk_one.py 8192 2048 2048 fwd 2>/dev/null | grep -v "^==" > gpurun_out/ncu_projfwd.csv
python - <<'P'
import csv
for f in ("gpurun_out/ncu_projdw.csv","gpurun_out/ncu_projfwd.csv"):
    rows=list(csv.DictReader(open(f)))
    out={}
    for r in rows: out.setdefault((r['ID'],r['Kernel Name'][:40]),{})[r['Metric Name']]=r['Metric Value']
    print(f)
    for k,v in out.items(): print(k, v)
P
