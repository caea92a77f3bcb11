import mmap, ctypes, os
libc = ctypes.CDLL("libc.so.6", use_errno=True)
n = 1 << 30
m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
print("madvise", libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(n), 14))  # MADV_HUGEPAGE
for i in range(0, n, 4096): m[i] = 1
for l in open("/proc/self/smaps_rollup"):
    if "AnonHuge" in l or l.startswith("Rss"): print(l.strip())
print([l.strip() for l in open("/proc/meminfo") if "Huge" in l])
