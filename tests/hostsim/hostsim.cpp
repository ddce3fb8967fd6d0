// TEST-ONLY host simulator: compiles the product's __host__ __device__ limb code
// (paper_2501_03245_b200/csrc/*.cuh) with g++ so that the exact device logic can be
// exercised in the GPU-less authoring container.  gecc_prims.cuh emulates the
// PTX carry flag on the host.  Nothing here is reachable from libgecc_b200.so.
#include <cstddef>
#include <cstdint>

#include "gecc_field.cuh"

using namespace gecc;

namespace {
fe col_get(const uint32_t* c, size_t n, size_t i) {
    fe v;
    for (int k = 0; k < 8; ++k) v.w[k] = c[k * n + i];
    return v;
}
void col_set(uint32_t* c, size_t n, size_t i, const fe& v) {
    for (int k = 0; k < 8; ++k) c[k * n + i] = v.w[k];
}

template <class F>
int field_op_t(const F& f, int op, size_t n, const uint32_t* a, const uint32_t* b, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) {
        fe x = col_get(a, n, i), y = b ? col_get(b, n, i) : fe_zero(), r = fe_zero();
        switch (op) {
            case 0: r = fe_mul(f, x, y); break;
            case 1: r = fe_add(f, x, y); break;
            case 2: r = fe_sub(f, x, y); break;
            case 3: r = fe_to_mont(f, x); break;
            case 4: r = fe_from_mont(f, x); break;
            case 5: r = fe_is_zero(x) ? x : fe_inv_fermat(f, x); break;
            case 6: r = fe_sqr(f, x); break;
            default: return 1;
        }
        col_set(out, n, i, r);
    }
    return 0;
}
}  // namespace

extern "C" {

// field: 0 SecpP 1 SecpN 2 Sm2P 3 Sm2N ; 4 = runtime field given by rt
int hs_field_op(int field, const FieldRT* rt, int op, size_t n, const uint32_t* a,
                const uint32_t* b, uint32_t* out) {
    switch (field) {
        case 0: return field_op_t(SecpP{}, op, n, a, b, out);
        case 1: return field_op_t(SecpN{}, op, n, a, b, out);
        case 2: return field_op_t(Sm2P{}, op, n, a, b, out);
        case 3: return field_op_t(Sm2N{}, op, n, a, b, out);
        case 4: return field_op_t(*rt, op, n, a, b, out);
    }
    return 1;
}

}  // extern "C"
