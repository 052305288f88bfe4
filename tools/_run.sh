timeout 120 python tools/sinr_once.py C3 8 > /dev/null && timeout 600 ncu --set full --import-source on --kernel-name regex:"k_small_grp" --launch-count 1 -o /tmp/sg -f timeout 300 python tools/sinr_once.py C3 8 > /dev/null 2>&1
python tools/ncu_lines.py /tmp/sg.ncu-rep 25 > gpurun_out/sg_lines.txt
ncu -i /tmp/sg.ncu-rep --page details --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
want=['Duration','Achieved Occupancy','Theoretical Occupancy','Compute (SM) Throughput','Executed Ipc Active','Issue Slots Busy','Registers Per Thread']
for r in rows[1:]:
    if r[mi] in want: print(r[mi], r[vi], r[ui])
" > gpurun_out/sg_details.txt
