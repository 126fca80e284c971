// Host run of the k_sparse_count8 list fill (c16_fill_group<4, true>, the code
// the setup kernel k_c16_fill runs per warp group) on lists read from a file;
// tools/c16_fill_sim.py writes the input and scores the output's shared-memory
// wavefronts per LDS.  Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//   --expt-relaxed-constexpr -Ipaper_2305_02510_b200/csrc -Iinclude tools/c16_fill_check.cu
#include "../paper_2305_02510_b200/csrc/k_sparse.cu"

#include <cstdio>
#include <vector>

namespace snb {
void launch_step_bump(int32_t*, cudaStream_t) {}  // not called; k_sparse.cu references it
}

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    int groups = 0;
    if (std::fread(&groups, 4, 1, f) != 1) return 2;
    const int nl = groups * 8;
    std::vector<uint2> desc(nl);
    std::vector<int64_t> off(nl + 1, 0);
    std::vector<uint32_t> meta;
    for (int p = 0; p < nl; ++p) {  // per post: descriptor word y, entry count, meta words
        uint32_t y = 0, n = 0;
        if (std::fread(&y, 4, 1, f) != 1 || std::fread(&n, 4, 1, f) != 1) return 2;
        std::vector<uint32_t> m(n);
        if (std::fread(m.data(), 4, n, f) != n) return 2;
        meta.insert(meta.end(), m.begin(), m.end());
        off[p + 1] = off[p] + n;
        desc[p].y = y;
    }
    std::fclose(f);
    uint64_t chunks = 0;
    for (int p = 0; p < nl; ++p) {
        if (p % 8 == 0)
            for (int q = p; q < p + 8; ++q) desc[q].x = static_cast<uint32_t>(chunks);
        chunks += desc[p].y >> 24;
    }
    std::vector<uint32_t> tmp(meta.size());
    std::vector<uint16_t> out(chunks * 8);
    for (int g = 0; g < groups; ++g)
        snb::c16_fill_group<4, true>(g, meta.data(), tmp.data(), off.data(), desc.data(), nl, 3 * 4095, out.data());
    FILE* o = std::fopen(argv[2], "wb");
    if (!o) return 2;
    std::fwrite(out.data(), 2, out.size(), o);
    std::fclose(o);
    return 0;
}
