import json,gzip,sys
t=json.load(gzip.open(sys.argv[1]))
ev=[e for e in t['traceEvents'] if e.get('ph')=='X' and e.get('cat') in ('kernel','gpu_memcpy')]
h2d=sorted([e for e in ev if 'HtoD' in e['name']],key=lambda e:e['ts'])
span=h2d[-1]['ts']+h2d[-1]['dur']-h2d[0]['ts']; busy=sum(e['dur'] for e in h2d)
gaps=[b['ts']-(a['ts']+a['dur']) for a,b in zip(h2d,h2d[1:])]
big=[g for g in gaps if g>20]
print('h2d busy %.1f ms of span %.1f ms (%.1f%%); gaps>20us: %d totalling %.2f ms; max %.0f us'%(busy/1e3,span/1e3,100*busy/span,len(big),sum(big)/1e3,max(gaps)))
