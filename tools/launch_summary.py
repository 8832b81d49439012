import csv, collections, sys
for fn in sys.argv[1:]:
    rows=[r for r in csv.reader(open(fn)) if len(r)>10]
    h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); mi=h.index('Metric Name'); idi=h.index('ID')
    per=collections.defaultdict(dict)
    for r in rows[1:]:
        per[(r[idi], r[ki].split('(')[0][-30:])][r[mi]]=(float(r[vi].replace(',','')), r[ui])
    agg=collections.defaultdict(lambda:[0,0.0,0.0,0.0,0.0])
    for (i,k),m in per.items():
        t=m['gpu__time_duration.sum']; v=t[0]/1e6 if t[1]=='ns' else (t[0]/1e3 if t[1]=='us' else t[0])
        a=agg[k]; a[0]+=1; a[1]+=v
        if 'smsp__thread_inst_executed_per_inst_executed.ratio' in m:
            a[2]+=m['smsp__thread_inst_executed_per_inst_executed.ratio'][0]*v; a[3]+=m.get('sm__warps_active.avg.pct_of_peak_sustained_active',(0,))[0]*v
        a.append(0) if len(a)<5 else None
        if 'dram__bytes_read.sum' in m:
            u={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
            a[4]+=m['dram__bytes_read.sum'][0]*u.get(m['dram__bytes_read.sum'][1],1)+m['dram__bytes_write.sum'][0]*u.get(m['dram__bytes_write.sum'][1],1)
    tot=sum(a[1] for a in agg.values())
    print(fn)
    for k,(c,v,lanes,wa,dr) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"  {k:32s} n={c:4d} {v:9.2f} ms {100*v/tot:5.1f}%  lanes={lanes/v if v else 0:5.1f} dram={dr/1e6:9.1f} MB")
