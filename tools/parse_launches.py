import csv,collections,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki,gi,mi,vi,ii=(h.index(x) for x in ("Kernel Name","Grid Size","Metric Name","Metric Value","ID"))
per=collections.defaultdict(dict); names={}
for r in rows[1:]:
    per[r[ii]][r[mi]]=float(r[vi].replace(',',''))
    names[r[ii]]=(r[ki].split('(')[0].replace('void ','').replace('hpg::',''),r[gi])
lim=int(sys.argv[2]) if len(sys.argv)>2 else 60
for i in sorted(per,key=int)[:lim]:
    m=per[i]; t=m['gpu__time_duration.sum']; b=m.get('dram__bytes_read.sum',0)+m.get('dram__bytes_write.sum',0)
    print(i,names[i][0][:40],names[i][1],f"{t/1e3:.1f}us {b/1e6:.1f}MB {b/t:.0f}GB/s hit {m.get('lts__t_sector_hit_rate.pct',0):.0f}%")
