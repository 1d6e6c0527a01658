#!/usr/bin/env python3
"""usage: sassmix.py OBJ KERNEL_SUBSTR -- instruction mix of each loop"""
import re,sys,subprocess,collections
obj,pat=sys.argv[1],sys.argv[2]
out=subprocess.run(['cuobjdump','-sass',obj],capture_output=True,text=True).stdout
funcs=re.split(r'\n\s+Function : ',out)
for f in funcs[1:]:
    name=f.split('\n',1)[0].strip()
    if pat not in name: continue
    ins=[]
    for l in f.splitlines():
        m=re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);',l)
        if m: ins.append((int(m.group(1),16),m.group(2)))
    print(name[:110],'total',len(ins))
    loops=[]
    for a,t in ins:
        m=re.search(r'BRA\S*\s+.*0x([0-9a-f]+)',t)
        if m and int(m.group(1),16)<a: loops.append((int(m.group(1),16),a))
    for lo,hi in loops:
        body=[t for a,t in ins if lo<=a<=hi]
        c=collections.Counter(re.sub(r'^@!?U?P\d+\s+','',t).split()[0].split('.')[0] for t in body)
        fp=sum(v for k,v in c.items() if k in('DADD','DMUL','DFMA'))
        print('  loop %x-%x n=%d fp64=%d other=%d'%(lo,hi,len(body),fp,len(body)-fp),{k:v for k,v in c.items() if k not in('DADD','DMUL','DFMA')})
