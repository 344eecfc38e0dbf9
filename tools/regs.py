"""Print registers / spills / stack per kernel from paper_1608_03630_b200/build.log (ptxas -v)."""
import re, sys
pat = sys.argv[1] if len(sys.argv) > 1 else ''
log = open('paper_1608_03630_b200/build.log').read().split('\n')
for i, l in enumerate(log):
    if 'Compiling entry function' in l and pat in l:
        name = re.search(r"'(.*)'", l).group(1)
        info = ' '.join(log[i + 1:i + 4])
        m = re.search(r'Used (\d+) registers', info); sp = re.search(r'(\d+) bytes spill stores', info)
        st = re.search(r'(\d+) bytes stack frame', info)
        print(name[:70].ljust(70), m and m.group(1), 'spill', sp and sp.group(1), 'stack', st and st.group(1))
