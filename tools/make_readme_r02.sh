# Regenerate README.md's generated status block (from "## Status (round 2" up to the NEXT-3 heading)
# out of profiles/r02_final (tools/readme_status_r02.py)
python3 - <<'PY'
import subprocess
s = open('README.md').read()
a = s.index('## Status (round 2')
b = s.index('### NEXT-3 (round 1 numbers')
gen = subprocess.run(['python', 'tools/readme_status_r02.py'], capture_output=True, text=True, check=True).stdout
s = s[:a] + "## Status (round 2, measured on one B200; every result bit-exact vs the oracle)\n\n" + gen + "\n\n" + s[b:]
open('README.md', 'w').write(s)
PY
