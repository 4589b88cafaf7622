// Exhaustive host check: closed-form probe count == the reference loop.
#include <cstdio>
#include "../paper_2111_08824_b200/csrc/lj_probe_count.h"
int main() {
    long checked = 0;
    for (int L = 1; L <= 70; ++L)
        for (int o = 0; o <= L; o += (L > 20 ? 7 : 1))
            for (int lb = 0; lb <= L; ++lb)
                for (int re = lb; re <= L; ++re)
                    for (int s = 0; s < L; ++s) {
                        int a = lj::ref_probe_count_loop(s - o, lb - o, re - o, L - o, -o);
                        int b = lj::ref_probe_count(s - o, lb - o, re - o, L - o, -o);
                        ++checked;
                        if (a != b) {
                            std::printf("MISMATCH L=%d o=%d lb=%d re=%d s=%d loop=%d fast=%d\n", L, o, lb, re, s, a, b);
                            return 1;
                        }
                    }
    // large distances
    for (int s = 0; s < 5000; s += 37)
        for (int lb = 0; lb < 70000; lb += 97)
            for (int run = 0; run < 40; run += 13) {
                int L = 1 << 17, re = lb + run;
                int a = lj::ref_probe_count_loop(s, lb, re, L, 0), b = lj::ref_probe_count(s, lb, re, L, 0);
                ++checked;
                if (a != b) { std::printf("MISMATCH2 s=%d lb=%d re=%d\n", s, lb, re); return 1; }
            }
    std::printf("OK %ld\n", checked);
    return 0;
}
