# usage: bash tools/spills.sh [extra nvcc flags]  -> spill instructions of the fused kernel by source line
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I/root/repo/include -lineinfo -cubin "$@" \
  -o /tmp/_sp.cubin /root/repo/paper_2506_06258_b200/csrc/fast.cu
nvdisasm -g /tmp/_sp.cubin > /tmp/_sp.dis
python3 - <<'PY'
import re,collections
cur=None; fn=None; cnt=collections.Counter()
for l in open('/tmp/_sp.dis'):
    m=re.match(r'\s*//## File ".*?fast.cu", line (\d+)',l)
    if m: cur=int(m.group(1)); continue
    m2=re.match(r'\s*\.text\.(\S+):',l)
    if m2: fn=m2.group(1)
    if fn and 'primal_fused' in fn and ('STL' in l or 'LDL' in l):
        cnt[(cur, 'STL' if 'STL' in l else 'LDL')]+=1
src=open('/root/repo/paper_2506_06258_b200/csrc/fast.cu').read().split('\n')
for k,v in sorted(cnt.items(), key=lambda kv: (kv[0][0] or 0)):
    print(k[0], k[1], v, src[k[0]-1].strip()[:80] if k[0] else '')
PY
