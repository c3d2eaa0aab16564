"""Print the SASS of one kernel (substring match), optionally a line range."""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
a = int(sys.argv[3]) if len(sys.argv) > 3 else 0
b = int(sys.argv[4]) if len(sys.argv) > 4 else 10**9
s = subprocess.check_output(["cuobjdump", "-sass", lib]).decode()
for f in re.split(r"\n\s*Function : ", s):
    name = f.split("\n")[0]
    if pat in name:
        n = 0
        for l in f.split("\n"):
            m = re.search(r"/\*([0-9a-f]{4})\*/\s+(.*?);", l)
            if m:
                if a <= n < b:
                    print(n, m.group(1), m.group(2))
                n += 1
        break
