/* ORACLE (test infrastructure only) — counter-based RNG, reading Q18.
 *
 * The paper draws random prolongation positions and random
 * visiting orders, but names no generator.  Both the oracle and the CUDA
 * path implement, independently, the same stateless generator so that their
 * random draws are bit-identical: the SplitMix64 output function
 *   mix(z) = let z += 0x9e3779b97f4a7c15;
 *            z = (z ^ z>>30) * 0xbf58476d1ce4e5b9;
 *            z = (z ^ z>>27) * 0x94d049bb133111eb;  z ^ z>>31
 * chained over (seed ^ purpose_tag, level, vertex*dim + comp). */
#include "mm_oracle.h"

uint64_t or_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

double or_uniform24(uint64_t key) {
    /* top 24 bits, scaled by 2^-24: exactly representable as float and double */
    return (double)(key >> 40) * (1.0 / 16777216.0);
}

uint64_t or_key_vertex(uint64_t seed, uint64_t tag, uint64_t level, uint64_t vertex, int dim, int comp) {
    uint64_t k = or_mix64(seed ^ tag);
    k = or_mix64(k ^ level);
    return or_mix64(k ^ (vertex * (uint64_t)dim + (uint64_t)comp));
}
