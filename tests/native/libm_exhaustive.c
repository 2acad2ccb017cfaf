// Exhaustive check of the device libm ports (paper_2405_07542_b200/csrc/
// glibc_mathf.h) against the HOST libm the reference links (glibc expf with
// its ifunc-selected variant, tanhf, expm1f).  Test infrastructure only.
//
//   libm_exhaustive [stride]   -> prints "<fn> <checked> <mismatches> <first bad bits>"
// stride 1 = all 2^32 inputs; larger strides sample every stride-th pattern.
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../paper_2405_07542_b200/csrc/glibc_mathf.h"

#define NT 8
typedef struct { uint64_t lo, hi, stride; uint64_t checked[3], bad[3]; uint32_t first[3]; } job_t;

static int same(float a, float b) {
    if (isnan(a) && isnan(b)) return 1;
    return sdm_f2u(a) == sdm_f2u(b);
}

static void* run(void* p) {
    job_t* j = (job_t*)p;
    for (int f = 0; f < 3; ++f) { j->checked[f] = 0; j->bad[f] = 0; j->first[f] = 0; }
    for (uint64_t u = j->lo; u < j->hi; u += j->stride) {
        float x = sdm_u2f((uint32_t)u);
        float a0 = expf(x), b0 = sd_expf(x);
        float a1 = tanhf(x), b1 = sd_tanhf(x);
        float a2 = expm1f(x), b2 = sd_expm1f(x);
        float as[3] = {a0, a1, a2}, bs[3] = {b0, b1, b2};
        for (int f = 0; f < 3; ++f) {
            j->checked[f]++;
            if (!same(as[f], bs[f])) {
                if (j->bad[f] == 0) j->first[f] = (uint32_t)u;
                j->bad[f]++;
            }
        }
    }
    return NULL;
}

int main(int argc, char** argv) {
    uint64_t stride = argc > 1 ? strtoull(argv[1], NULL, 10) : 1;
    pthread_t th[NT];
    job_t jobs[NT];
    uint64_t total = 1ull << 32, chunk = total / NT;
    for (int t = 0; t < NT; ++t) {
        jobs[t].lo = chunk * t;
        jobs[t].hi = chunk * (t + 1);
        jobs[t].stride = stride;
        pthread_create(&th[t], NULL, run, &jobs[t]);
    }
    const char* names[3] = {"expf", "tanhf", "expm1f"};
    uint64_t checked[3] = {0}, bad[3] = {0};
    uint32_t first[3] = {0};
    int have[3] = {0};
    for (int t = 0; t < NT; ++t) {
        pthread_join(th[t], NULL);
        for (int f = 0; f < 3; ++f) {
            checked[f] += jobs[t].checked[f];
            if (jobs[t].bad[f] && !have[f]) { first[f] = jobs[t].first[f]; have[f] = 1; }
            bad[f] += jobs[t].bad[f];
        }
    }
    for (int f = 0; f < 3; ++f)
        printf("%s %llu %llu 0x%08x\n", names[f], (unsigned long long)checked[f],
               (unsigned long long)bad[f], first[f]);
    return (bad[0] || bad[1] || bad[2]) ? 1 : 0;
}
