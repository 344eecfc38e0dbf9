#!/bin/bash
# Instruction histogram of one kernel's SASS: tools/sass_fn.sh LIB FUNC_SUBSTRING [N]
awk -v pat="$2" '/Function : /{p = index($0, pat) > 0} p' <(cuobjdump -sass "$1") > /tmp/fn.sass
grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[T0-9] )?[A-Z0-9_.]+" /tmp/fn.sass | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -${3:-25}
