# ptxas spill / stack summary of engine.cu's device functions (no link): bash tools/probes/ptxas_stats.sh [-Dflags]
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -ccbin /usr/bin/g++ -lineinfo "$@" -Xptxas -v -c paper_1812_06635_b200/csrc/engine.cu -o /dev/null 2>&1 | python3 -c "
import sys,re
name=None
for ln in sys.stdin:
    m=re.search(r'Function properties for (\S+)',ln)
    if m:
        name=re.sub(r'^_ZN\d+_INTERNAL_\w+?GLOBAL__N__\w+?cu_\d+','',m.group(1))[:40]; continue
    if 'spill' in ln and name:
        print(name, '|', ln.strip()); name=None
"
