#!/bin/bash
# SASS evidence for profiles/: opcode histogram of one kernel of a built object + the lines that prove the
# asynchronous-copy / mbarrier / 128-bit-atomic / wide-multiply design.  Runs here (no GPU needed).
#   scripts/sass_excerpt.sh <object> <mangled-name-substring> > profiles/<file>
obj=$1; fn=$2
cuobjdump -sass "$obj" | awk -v fn="$fn" '
  /Function :/ { on = index($0, fn) > 0; if (on) print "## " $0 }
  on && /^ +\/\*[0-9a-f]+\*\/ +[A-Z@]/ { print }
' > /tmp/sass_fn.txt
echo "# $(basename $obj): $(grep -vc '^## ' /tmp/sass_fn.txt) SASS instructions in $(grep -c '^## ' /tmp/sass_fn.txt) function(s) matching '$fn'"
grep '^## ' /tmp/sass_fn.txt
echo "# arch: $(cuobjdump -lelf "$obj" | head -3 | tr '\n' ' ')"
echo "# opcode histogram (top 24)"
grep -v '^## ' /tmp/sass_fn.txt | sed -E 's/^ +\/\*[0-9a-f]+\*\/ +//; s/^@!?U?P[0-9T]+ +//' | awk '{print $1}' | sed 's/;$//' | sort | uniq -c | sort -rn | head -24
for pat in 'UBLKCP' 'SYNCS' 'LDGSTS' 'ATOMG.E.CAS.128' 'ATOMG.E.MIN' 'IMAD.WIDE.U32' 'LEA.HI' 'UTMALDG|UTCMMA|UTCHMMA|LDTM|HMMA'; do
  n=$(grep -E -c "$pat" /tmp/sass_fn.txt)
  echo "# $pat: $n line(s); first three:"
  grep -E -m3 "$pat" /tmp/sass_fn.txt | sed -E 's/ +/ /g'
done
