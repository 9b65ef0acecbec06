"""Apply one block once (ncu capture helper): python tools/one_block.py N CHUNK 'G1;G2;...'"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n, chunk = int(sys.argv[1]), int(sys.argv[2])
lines = [g.strip() for g in sys.argv[3].split(";") if g.strip()]
st = qk.State(n)
qk.apply_block(st, lines, chunk)
qk.apply_block(st, lines, chunk)
