"""Opcode mix of k_classify<false>'s dense loop (from the first FMUL2 back 50 to the first REDUX.OR)."""
import re, subprocess, sys
from collections import Counter
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1912_11494_b200/libsegb200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blk = out.split("Function : _ZN3seg10k_classifyILb0ELb0EEEvNS_14ClassifyParamsE")[1].split("Function :")[0]
ins = [m.group(1).strip() for m in re.finditer(r'/\*[0-9a-f]+\*/\s+(.*?);', blk)]
ri = [k for k, t in enumerate(ins) if 'REDUX.OR' in t][0]
fi = [k for k, t in enumerate(ins) if 'FMUL2' in t][0]
seg = ins[max(0, fi - 50):ri + 1]
c = Counter(t.split()[1] if t.startswith('@') else t.split()[0] for t in seg)
print(len(seg), c.most_common(20))
