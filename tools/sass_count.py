"""Per-function SASS opcode histogram of a `cuobjdump -sass` dump (authoring aid).
Non-inlined device functions live inside the kernel's code: they are found as CALL
targets and run to the next RET.   usage: sass_count.py dump.sass [kernel-regex]"""
import re, collections, sys

kern = None
code = collections.defaultdict(list)   # kernel -> [(addr, op, full)]
for l in open(sys.argv[1]):
    m = re.search(r'Function : (\S+)', l)
    if m:
        kern = m.group(1)
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,6})\*/\s+(@!?U?P\d\s+)?([A-Z0-9_.]+)(.*?);', l)
    if m and kern:
        code[kern].append((int(m.group(1), 16), m.group(3), m.group(4)))

def base(op):
    return '.'.join(op.split('.')[:2]) if op.startswith('IMAD') else op.split('.')[0]

pat = sys.argv[2] if len(sys.argv) > 2 else '.'
for k, ins in code.items():
    if not re.search(pat, k):
        continue
    targets = collections.Counter()
    for a, op, rest in ins:
        if op.startswith('CALL'):
            m = re.search(r'0x([0-9a-f]+)', rest)
            if m:
                targets[int(m.group(1), 16)] += 1
    print(k[:110], 'instructions:', len(ins))
    for t, ncalls in sorted(targets.items()):
        c = collections.Counter()
        n = 0
        for a, op, rest in ins:
            if a < t:
                continue
            c[base(op)] += 1
            n += 1
            if op.startswith('RET'):
                break
        print('   callee @0x%x (%d call sites): %d instr' % (t, ncalls, n), dict(c.most_common()))
