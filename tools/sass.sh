#!/bin/bash
# tools/sass.sh <object> <mangled-function> <out>: clean SASS listing of one kernel + (line, #VIMNMX3) of every loop body
cuobjdump -sass -fun "$2" "$1" | grep -v "^\s*/\* 0x" | sed 's/\/\*[0-9a-f]\{4,5\}\*\///' | sed 's/\s*\/\* 0x[0-9a-f]* \*\///' > "$3"
wc -l "$3"
awk '/VIMNMX3/{c++} /BRA/{ if(c>0) print NR, c; c=0}' "$3" | head -${4:-12}
