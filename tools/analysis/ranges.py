import re
def ranges(path='/root/repo/paper_2310_17274_b200/csrc/crb_device.cuh'):
    L = open(path).read().split('\n')
    def find(pat, start=0):
        for i in range(start, len(L)):
            if re.search(pat, L[i]): return i + 1
        raise KeyError(pat)
    m = {}
    m['fk_chain'] = find(r'^__device__ __forceinline__ void fk_chain')
    m['place'] = find(r'^__device__ __forceinline__ void fk_place')
    m['sweep'] = find(r'^// Sweep directions of sphere')
    m['box_slow_end'] = find(r'^// One evaluation pass over the 32 slots')
    m['a2'] = find(r'// ---- a2:')
    m['a3'] = find(r'// ---- a3:')
    m['a7'] = find(r'// ---- a7:')
    m['a4'] = find(r'// ---- a4 \+ a5')
    m['exact'] = find(r'auto exact_box = ')
    m['wscreen'] = find(r'if \(__any_sync\(FULL, th2\[0\] > 0.f')
    m['wepi'] = find(r"the group's cost goes to the")
    m['self'] = find(r'const uint4 B = blk\[item - nwg\]')
    m['a10'] = find(r'// ---- a10')
    m['a9'] = find(r'// ---- a9:')
    m['jg'] = find(r'// joint gradient: the subtree')
    m['tr'] = find(r'// ---- transposed stencil')
    m['end'] = find(r'^__device__ __forceinline__ float pass_gdot')
    R = [("fk_chain", m['fk_chain'], m['place'] - 1), ("place", m['place'], m['place'] + 40),
         ("box_slow+helpers", m['sweep'], m['box_slow_end'] - 1), ("a2", m['a2'], m['a3'] - 1),
         ("a8", m['a3'], m['a7'] - 1), ("pose", m['a7'], m['a4'] - 1), ("wsetup", m['a4'], m['exact'] - 1),
         ("exact_box", m['exact'], m['wscreen'] - 1), ("wscreen", m['wscreen'], m['wepi'] - 1),
         ("wepi", m['wepi'], m['self'] - 1), ("self", m['self'], m['a10'] - 1), ("merge", m['a10'], m['a9'] - 1),
         ("linksums", m['a9'], m['jg'] - 1), ("jointgrad", m['jg'], m['tr'] - 1), ("transposed", m['tr'], m['end']),
         ("misc_hdr", 1, m['fk_chain'] - 1)]
    return R
