# usage: tools/regs.sh fill_s16  -> instance, registers, spill bytes
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Iinclude -Ipaper_2002_04561_b200/csrc -Xptxas -v -c paper_2002_04561_b200/csrc/$1.cu -o /tmp/x.o 2>&1 | python3 -c "
import sys, re
cur = None
for line in sys.stdin:
    m = re.search(r\"Compiling entry function '(\S+)'\", line)
    if m: cur = m.group(1).replace('_ZN6anyseq11fill_kernelI','').replace('EEEvNS_8FillArgsE',''); continue
    m = re.search(r'(\d+) bytes spill stores', line)
    if m: sp = m.group(1)
    m = re.search(r'Used (\d+) registers', line)
    if m and cur: print(cur, 'regs', m.group(1), 'spill', sp); cur = None
"
