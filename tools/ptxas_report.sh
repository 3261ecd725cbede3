#!/bin/bash
# registers / stack per kernel (same flags as build.py)
cd "$(dirname "$0")/../paper_1609_04471_b200"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared --expt-relaxed-constexpr -Xptxas -v -o /tmp/ptxas_probe.so csrc/sr_sort.cu 2>&1 | python3 -c "
import sys,re,subprocess
cur=None
for line in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: cur=subprocess.run(['c++filt',m.group(1)],capture_output=True,text=True).stdout.strip()[:70]; continue
    if 'error' in line: print(line.strip()[:200]); continue
    m=re.search(r'(\d+) bytes stack frame',line)
    if m and cur: st=int(m.group(1))
    m=re.search(r'Used (\d+) registers',line)
    if m and cur: print(f'{m.group(1):>4} regs stack={st:<4} {cur}'); cur=None
" | sort -k4 | uniq | head -${1:-80}
