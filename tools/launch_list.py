"""Per-launch time and DRAM bytes of an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).
usage: launch_list.py launches.csv [last_n]"""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if r and r[0]=='ID': hdr=r; start=i; break
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
data=collections.defaultdict(dict)
for r in rows[start+1:]:
    if len(r)<len(hdr): continue
    data[int(r[ii])][r[mi]]=(r[ki], r[vi])
items=sorted(data.items())
n=int(sys.argv[2]) if len(sys.argv)>2 else 40
for id_, d in items[-n:]:
    name=list(d.values())[0][0][:60]
    t=float(d['gpu__time_duration.sum'][1].replace(',',''))
    rd=float(d['dram__bytes_read.sum'][1].replace(',','')); wr=float(d['dram__bytes_write.sum'][1].replace(',',''))
    print(f"{id_:4d} {t/1e3:9.1f} us  rd {rd/1e9:6.2f} wr {wr/1e9:6.2f}  {name}")
