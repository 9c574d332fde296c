"""Static check of the contraction's SASS: distance (in DMMA instructions)
between a DMMA and the next DMMA consuming its accumulator.  Short chains
show up as 'stall_wait' (fixed-latency dependency) in ncu."""
import re, subprocess, sys, collections

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1605_01584_b200/lib/libpcc_b200.so"
fn = sys.argv[2] if len(sys.argv) > 2 else "syrk_kernelILi0E"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", sass)
for b in blocks:
    if fn not in b.split("\n")[0]:
        continue
    d = [l for l in b.split("\n") if "DMMA" in l]
    seq = []
    for l in d:
        m = re.search(r"DMMA\.8x8x4 R(\d+), R(\d+), R(\d+), R(\d+)", l)
        if m:
            seq.append(tuple(int(v) for v in m.groups()))
    last_write = {}
    dist = collections.Counter()
    for i, (dst, a, bb, c) in enumerate(seq):
        if c in last_write:
            dist[i - last_write[c]] += 1
        last_write[dst] = i
    print(b.split("\n")[0][:80], "DMMAs:", len(seq), "chain distance histogram:", sorted(dist.items()))
