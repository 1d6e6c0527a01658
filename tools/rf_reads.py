#!/usr/bin/env python3
"""usage: rfreads.py OBJ KERNEL_SUBSTR -- RF register-pair reads per FP64 instruction of the largest innermost loop, counting operand-reuse hits"""
import re,collections,subprocess,sys
obj,pat=sys.argv[1],sys.argv[2]
out=subprocess.run(['cuobjdump','-sass',obj],capture_output=True,text=True).stdout
for f in re.split(r'\n\s+Function : ',out)[1:]:
    name=f.split('\n',1)[0].strip()
    if pat not in name: continue
    ins=[]
    for l in f.splitlines():
        m=re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);',l)
        if m: ins.append((int(m.group(1),16),m.group(2).strip()))
    loops=[]
    for a,t in ins:
        m=re.search(r'BRA\S*\s+.*0x([0-9a-f]+)',t)
        if m and int(m.group(1),16)<a: loops.append((int(m.group(1),16),a))
    inner=[(lo,hi) for lo,hi in loops if not any((l2>=lo and h2<=hi) and (l2,h2)!=(lo,hi) for l2,h2 in loops)]
    lo,hi=max(inner,key=lambda x:x[1]-x[0])
    body=[t for a,t in ins if lo<=a<=hi]
    def parse(t):
        t=re.sub(r'^@!?U?P\d+\s+','',t)
        parts=t.split(None,1)
        if len(parts)<2: return parts[0],[]
        return parts[0],[x.strip() for x in parts[1].split(',')][1:]
    norm=lambda x: re.sub(r'[-|]|\.reuse','',x)
    stat=collections.Counter(); prev=None
    for t in body:
        op,s=parse(t)
        if op.startswith(('DFMA','DADD','DMUL')):
            fed=0
            if prev:
                for i,x in enumerate(s):
                    if i<len(prev[1]) and '.reuse' in prev[1][i] and norm(prev[1][i])==norm(x): fed+=1
            stat[(op.split('.')[0],len(set(map(norm,s)))-fed)]+=1
        prev=(op,s)
    print(name[:90]); print(' loop',hex(lo),hex(hi),len(body),sorted(stat.items()))
    cyc=sum(max(2,k[1])*v for k,v in stat.items()); n=sum(stat.values())
    print(' fp64 instr',n,'RF-limited cycles',cyc,'ratio',cyc/(2*n))
