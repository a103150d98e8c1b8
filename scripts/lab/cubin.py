"""Minimal ELF64 cubin access for SASS experiments: find a kernel's .text section,
iterate its 128-bit instructions, and rewrite fields in place.

Field layout of the 3-source ALU form (Volta..Blackwell, checked against cuobjdump
-sass on sm_100a): opcode bits 0-11, Rd 16-23, Ra 24-31, Rb 32-39, Rc 64-71;
control: stall 105-108, yield 109, write barrier 110-112, read barrier 113-115,
wait mask 116-121, reuse flags 122-125 (A, B, C, ... slot bits)."""
import struct


class Cubin:
    def __init__(self, path):
        self.data = bytearray(open(path, "rb").read())
        d = self.data
        assert d[:4] == b"\x7fELF" and d[4] == 2, "not an ELF64 cubin"
        shoff, = struct.unpack_from("<Q", d, 0x28)
        shentsize, shnum, shstrndx = struct.unpack_from("<HHH", d, 0x3A)
        secs = []
        for i in range(shnum):
            name, typ, flags, addr, off, size = struct.unpack_from("<IIQQQQ", d, shoff + i * shentsize)
            secs.append((name, off, size))
        stroff = secs[shstrndx][1]
        self.sections = {}
        for name, off, size in secs:
            end = d.index(b"\0", stroff + name)
            self.sections[d[stroff + name:end].decode()] = (off, size)

    def text(self, kernel):
        return self.sections[".text." + kernel]

    def insn(self, kernel, pc):
        off, size = self.text(kernel)
        assert 0 <= pc < size and pc % 16 == 0
        lo, hi = struct.unpack_from("<QQ", self.data, off + pc)
        return lo | (hi << 64)

    def set_insn(self, kernel, pc, v):
        off, _ = self.text(kernel)
        struct.pack_into("<QQ", self.data, off + pc, v & (2**64 - 1), v >> 64)

    def save(self, path):
        open(path, "wb").write(self.data)


def field(v, lo, n):
    return (v >> lo) & ((1 << n) - 1)


def set_field(v, lo, n, x):
    m = ((1 << n) - 1) << lo
    return (v & ~m) | ((x << lo) & m)


OPC_DFMA_RRR = 0x22B  # DFMA Rd, Ra, Rb, Rc (all registers)
