// ABI plumbing: error reporting, host-memory mapping, PCG64 jump tables.
#include "common.cuh"
#include "pcg64.cuh"

namespace bgl {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// One thread per batch: row 0 = stream state; rows 1..64 = 2^k-step maps.
__global__ void pcg64_tables_kernel(const uint64_t* __restrict__ states, int64_t nb,
                                    uint64_t* __restrict__ tables) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const uint64_t* s = states + 4 * b;
    uint64_t* t = tables + 65 * 4 * b;
    t[0] = s[0];
    t[1] = s[1];
    t[2] = s[2];
    t[3] = s[3];
    U128 A{2549297995355413924ull, 4865540595714422341ull};
    U128 C{s[2], s[3]};
    const U128 one{0, 1};
    for (int k = 0; k < 64; ++k) {
        uint64_t* r = t + 4 * (1 + k);
        r[0] = A.hi;
        r[1] = A.lo;
        r[2] = C.hi;
        r[3] = C.lo;
        C = mul128(add128(A, one), C);
        A = mul128(A, A);
    }
}

__global__ void pcg64_draws_kernel(const uint64_t* __restrict__ table, int64_t first, int64_t n,
                                   uint64_t* __restrict__ out) {
    PcgTable T{table};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = draw_of_state(T.at((uint64_t)(first + i + 1)));
}

}  // namespace bgl

using namespace bgl;

extern "C" {

const char* bgl_last_error(void) { return g_err; }

int bgl_abi_version(void) { return 1; }

int bgl_host_device_pointer(void* host_ptr, void** dev_ptr) {
    BGL_CHECK_ARG(host_ptr && dev_ptr, "bgl_host_device_pointer: null pointer");
    return cuda_status(cudaHostGetDevicePointer(dev_ptr, host_ptr, 0), "cudaHostGetDevicePointer");
}

int bgl_host_register(void* host_ptr, size_t bytes) {
    BGL_CHECK_ARG(host_ptr && bytes, "bgl_host_register: empty buffer");
    return cuda_status(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable),
                       "cudaHostRegister");
}

int bgl_host_unregister(void* host_ptr) {
    return cuda_status(cudaHostUnregister(host_ptr), "cudaHostUnregister");
}

int bgl_pcg64_tables(const uint64_t* states, int64_t nb, uint64_t* tables, void* stream) {
    BGL_CHECK_ARG(nb >= 0, "bgl_pcg64_tables: nb < 0");
    if (nb == 0) return BGL_OK;
    BGL_CHECK_ARG(states && tables, "bgl_pcg64_tables: null pointer");
    pcg64_tables_kernel<<<(unsigned)ceil_div(nb, 128), 128, 0, as_stream(stream)>>>(states, nb, tables);
    return launch_status("pcg64_tables_kernel");
}

int bgl_pcg64_draws(const uint64_t* table, int64_t first, int64_t n, uint64_t* out, void* stream) {
    BGL_CHECK_ARG(first >= 0 && n >= 0, "bgl_pcg64_draws: negative range");
    if (n == 0) return BGL_OK;
    pcg64_draws_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(table, first, n, out);
    return launch_status("pcg64_draws_kernel");
}

}  // extern "C"
